# bench + launch list + one full ncu capture of the dense solver; summaries go to profiles/
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_solve_dense -c 1 -o gpurun_out/dense_final -f python tools/profile_dense.py --iters 100 > gpurun_out/ncu_final.log 2>&1
echo done
