mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -8 > gpurun_out/pytest_gpu.log
python tools/profile_dense.py --iters 100 --reps 3 > gpurun_out/prof_plain.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_solve_dense -c 1 -o gpurun_out/dense_k100 -f python tools/profile_dense.py --iters 100 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_ncu.log 2>&1
tail -3 gpurun_out/ncu1.log
