set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -5 gpurun_out/smoke.log
LSK_CPU_ITERS=2 timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; tail -3 gpurun_out/bench.log
