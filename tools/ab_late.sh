for i in 1 2; do
  for lib in "" "$PWD/_ab/late.so"; do
    echo "== ${lib##*/}"
    NQKV_LIB=$lib timeout 600 python tools/ragged_probe.py 2>&1 | grep "fused=1"
    for wl in c5 c2 c4; do
      echo "$wl $(NQKV_LIB=$lib timeout 400 python bench.py --workload $wl --no-configs --no-cpu-baseline --steps 20 2>/dev/null | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['roofline']['mean_launch_us'],2), d['clocks']['sm_mhz'])")"
    done
  done
done
