# full round check on a gpurun box: GPU tests, the default bench line, its ncu launch list, sharded-design timings
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $? $(tail -1 gpurun_out/pytest_gpu.log)"
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/bench_full.log > gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/bench_ncu.log 2>&1; echo "ncu rc $?"
timeout 900 python tools/profile_sharded.py > gpurun_out/sharded.md 2>&1; echo "sharded rc $?"; cat gpurun_out/sharded.md
