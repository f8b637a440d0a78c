# two-team dense kernel: timing A/B against the one-team kernel, parity, short bench
mkdir -p gpurun_out
for n in 1184 8192; do for t in "" "--one-team"; do echo "n=$n $t"; timeout 120 python tools/profile_dense.py --n $n --iters 200 --reps 3 $t; done; done > gpurun_out/teams_prof.log 2>&1
cat gpurun_out/teams_prof.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py tests/test_gpu_fuzz.py -x -q -p no:cacheprovider > gpurun_out/teams_pytest.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/teams_pytest.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-extra > gpurun_out/teams_bench.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/teams_bench.log | cut -c1-300
