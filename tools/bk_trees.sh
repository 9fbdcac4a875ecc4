# tools/bench_kernels.py (c1, c2) for the working tree and the trees under _ab/t_*, interleaved
for i in 1 2; do for d in . _ab/t_*; do
  (cd $d && timeout 120 python tools/bench_kernels.py --configs c1,c2 2>&1 | sed "s|^|$d |")
done; done
