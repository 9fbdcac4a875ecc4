#!/bin/bash
# Run on the GPU box (gpurun): the bench, the ncu launch list of the same
# bench command, and one `ncu --set full` capture each of the decode and bulk
# quantize kernels (each ncu command is preceded by the identical plain run).
set -u
R=${1:-r1}
O=gpurun_out
mkdir -p $O
CMD="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-configs"
$CMD > $O/${R}_bench_small_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|quantize_kernel" --csv --log-file $O/${R}_launches.csv $CMD > $O/${R}_launches_run.log 2>&1
$CMD > $O/${R}_bench_small_plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 100 -c 1 -o $O/${R}_decode $CMD > $O/${R}_ncu_decode.log 2>&1
$CMD > $O/${R}_bench_small_plain3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:quantize_kernel -s 2 -c 1 -o $O/${R}_quantize $CMD > $O/${R}_ncu_quant.log 2>&1
ls -la $O | tail -20
# prefill (c4 prompt, tools/prefill_one.py): plain run, then one full capture
python tools/prefill_one.py > $O/${R}_prefill_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 1 -c 1 -o $O/${R}_prefill python tools/prefill_one.py > $O/${R}_ncu_prefill.log 2>&1
