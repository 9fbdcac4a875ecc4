# A/B of bench.py ms_per_step (interleaved runs): env var $1 with values 1 / 0
for i in 1 2; do for v in 1 0; do
  r=$(env $1=$v python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['mean_launch_us'])")
  echo "$1=$v $r"
done; done
