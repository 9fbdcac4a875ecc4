# A/B of bench.py ms_per_step over several library builds (NQKV_LIB), interleaved,
# plus the _ab/head tree if present:  bash tools/ab_libs.sh lib1.so lib2.so ...
for i in 1 2; do
  for lib in "" "$@"; do
    r=$(NQKV_LIB=$lib python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['mean_launch_us'])")
    echo "${lib:-in-tree} $r"
  done
  if [ -d _ab/head ]; then
    r=$(cd _ab/head && python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['mean_launch_us'])")
    echo "head $r"
  fi
done
