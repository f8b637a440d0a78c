for n in 148 1184 8192; do echo "n=$n $(timeout 120 python tools/profile_dense.py --n $n --m 8192 --iters 200 --reps 3 | tail -1)"; done
echo "check1000 $(timeout 120 python tools/profile_dense.py --n 8192 --iters 200 --reps 3 --check 1000 | tail -1)"
LSK_PARITY_LOG=gpurun_out/parity_ap.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py tests/test_gpu_fuzz.py tests/test_gpu_cluster.py -q -p no:cacheprovider 2>&1 | tail -3
