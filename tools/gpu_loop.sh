# dense m > 8192 loop: timing and the tests that cover its kernels and the half-step API
for a in "--n 16384 --m 16384" "--n 16384 --m 16384 --general" "--n 8192 --m 16384" "--n 4096 --m 32768"; do
  echo "[$a] $(timeout 300 python tools/profile_dense.py $a --iters 50 --reps 2 2>&1 | tail -1)"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz_halfsteps.py tests/test_gpu_fuzz.py -q -p no:cacheprovider 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -c 60 --csv --log-file gpurun_out/loop_launches.csv python tools/profile_dense.py --n 16384 --m 16384 --iters 10 --reps 1 > /dev/null 2>&1; echo "ncu rc $?"
