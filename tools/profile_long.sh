#!/bin/bash
# Steady-state ncu captures (one sequence per CTA): decode at hd 64 and hd 128,
# each preceded by the identical plain run; summaries written to gpurun_out/.
R=${1:-r1i}
O=gpurun_out
for cfg in "1 148 64 16384" "1 148 128 8192"; do
  tag=long$(echo $cfg | cut -d' ' -f3)
  python tools/long_case.py $cfg 1 > $O/${R}_${tag}_plain.log 2>&1 && \
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_kernel -c 1 \
      -o $O/${R}_${tag} python tools/long_case.py $cfg 1 > $O/${R}_${tag}_ncu.log 2>&1
  (echo "# ncu --set full, steady state: tools/long_case.py $cfg (one sequence per CTA, 174.6 MB, 1 launch, cold L2)"
   python tools/ncu_summary.py $O/${R}_${tag}.ncu-rep 2>&1 | grep -E "Duration|Throughput|Ipc|Issue Slots|Eligible|Registers|Shared Memory Per Block" | sed 's/  */ /g'
   ncu -i $O/${R}_${tag}.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[-1]
keys=['l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','dram__bytes_read.sum','smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active','smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active','smsp__average_warps_issue_stalled_wait_per_issue_active','smsp__average_warps_issue_stalled_selected_per_issue_active']
for k,x in zip(h,v):
  if any(k.startswith(s) for s in keys): print('raw',k,x)
") > $O/${R}_decode_${tag}_ncu.txt
  rm -f $O/${R}_${tag}.ncu-rep
done
