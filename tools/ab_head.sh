# A/B of bench.py ms_per_step: working tree (optionally under env $AB_ENV) vs
# a copy of another commit's tree built under _ab/head (untracked), interleaved.
for i in 1 2; do for d in . _ab/head; do
  r=$(cd $d && env $AB_ENV python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['mean_launch_us'])")
  echo "$d $r"
done; done
