set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2d_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2d_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2d_bench.log 2>&1; echo "bench rc $?" >> gpurun_out/r2d_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2d_ref.log 2>&1
