mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "taskq" 2>&1 | tail -15 > gpurun_out/pytest_v4.log
for n in 148 1184 8192; do python tools/profile_dense.py --n $n --iters 200 --reps 3 --taskq; done > gpurun_out/prof_v4.log 2>&1
cat gpurun_out/pytest_v4.log gpurun_out/prof_v4.log
