# Round-end evidence on the GPU box: GPU suite, smoke, bench (both arms),
# launch list + ncu captures (tools/profile_round.sh), csv pages only.
set -u
R=${1:-r2e}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/${R}_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${R}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${R}_bench.log 2>&1; echo "bench rc $?" >> gpurun_out/${R}_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_ref.log 2>&1
timeout 1200 bash tools/profile_round.sh ${R} > gpurun_out/${R}_profile.log 2>&1
bash tools/profile_shrink.sh >> gpurun_out/${R}_profile.log 2>&1
