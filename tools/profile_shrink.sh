#!/bin/bash
# On the GPU box after tools/profile_round.sh: turn each .ncu-rep under
# gpurun_out/ into csv pages (details, raw, sass source) and delete the
# report, so the results fit gpurun's 64 MiB copy-back limit.
for rep in gpurun_out/*.ncu-rep; do
  [ -e "$rep" ] || continue
  b=${rep%.ncu-rep}
  ncu -i "$rep" --page details --csv > ${b}_details.csv 2>/dev/null
  ncu -i "$rep" --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i "$rep" --page source --csv --print-source sass > ${b}_sass.csv 2>/dev/null
  rm -f "$rep"
done
du -sh gpurun_out
