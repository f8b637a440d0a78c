# full bench + launch list of the same command (ncu, cold-cache serialised)
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/bench_ncu.log 2>&1
echo launches $(grep -c . gpurun_out/launches.csv)
