#!/bin/bash
# Run on the GPU box: one `ncu --set full` capture of the decode (attend) and
# bulk quantize kernels for each of c3, c4, c5 (one layer; c5 at the 12-head
# shard), each preceded by the identical plain run.
set -u
R=${1:-r1f}
O=gpurun_out
mkdir -p $O
for c in c3 c4 c5; do
  for k in attend quantize; do
    CMD="python tools/bench_kernels.py --configs $c --only $k ${BLK:+--blk $BLK}"
    kern=$([ $k = attend ] && echo decode_kernel || echo quantize_kernel)
    skip=$([ $k = attend ] && echo 1 || echo 0)
    timeout 300 $CMD > $O/${R}_${c}_${k}_plain.log 2>&1 && \
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kern -s $skip -c 1 \
        -o $O/${R}_${c}_${k} $CMD > $O/${R}_${c}_${k}_ncu.log 2>&1
  done
done
ls $O | grep "^${R}_c" | head -30
