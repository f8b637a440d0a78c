# m <= 1024 cluster solvers (single cluster, multi-cluster): timing vs the grid solver, parity tests
mkdir -p gpurun_out
for a in "--n 16 --m 1024" "--n 128 --m 1024" "--n 256 --m 1024" "--n 256 --m 1024 --no-cluster" "--n 512 --m 1024" "--n 512 --m 1024 --no-cluster" "--n 1024" "--n 1024 --no-cluster" "--n 1024 --check 1000" "--n 2048 --m 1024" "--n 2048 --m 1024 --no-cluster" "--n 4096 --m 1024" "--n 4096 --m 1024 --no-cluster" "--n 8192 --m 1024" "--n 8192 --m 1024 --no-cluster"; do
  echo "[$a] $(timeout 120 python tools/profile_dense.py $a --eps 1e-2 --iters 200 --reps 3 2>&1 | tail -1)"
done > gpurun_out/c1.log 2>&1; cat gpurun_out/c1.log
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -4 gpurun_out/smoke.log
if [ "${FULL:-1}" = "1" ]; then timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "FAILED|passed|failed|Error" gpurun_out/pytest_gpu.log | tail -15; fi
