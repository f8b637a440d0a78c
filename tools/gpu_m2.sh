for lib in paper_2605_00837_b200/liblsk.so build/liblsk_mult1.so; do for n in 1184 8192; do echo "$lib n=$n $(LSK_LIB=$lib timeout 120 python tools/profile_dense.py --n $n --m 8192 --iters 200 --reps 3 2>&1 | tail -1)"; done; done
echo "m4096 $(timeout 120 python tools/profile_dense.py --n 8192 --m 4096 --iters 200 --reps 3 | tail -1)"
echo "m4096 mult1 $(LSK_LIB=build/liblsk_mult1.so timeout 120 python tools/profile_dense.py --n 8192 --m 4096 --iters 200 --reps 3 | tail -1)"
LSK_PARITY_LOG=gpurun_out/parity_m2.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_long.py tests/test_gpu_fuzz.py tests/test_gpu_cluster.py -q -p no:cacheprovider 2>&1 | tail -3
