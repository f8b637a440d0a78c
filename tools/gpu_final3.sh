# end-of-round check (late round 2, direct arithmetic by default): tests (+ parity log), smoke, bench +
# launch list, one ncu --set full capture of the dense kernel at C2 (DRAM traffic for roofline.traffic)
mkdir -p gpurun_out
rm -f gpurun_out/parity_errors.jsonl
LSK_PARITY_LOG=$PWD/gpurun_out/parity_errors.jsonl timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $? $(tail -1 gpurun_out/pytest_gpu.log)"; grep FAILED gpurun_out/pytest_gpu.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -4 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/bench_full.log > gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/bench_ncu.log 2>&1; echo "ncu rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_solve_dense -c 1 -o gpurun_out/dense_r2direct -f python tools/profile_dense.py --iters 100 > gpurun_out/ncu_direct.log 2>&1; echo "ncu full rc $?"
python tools/ncu_summary.py gpurun_out/dense_r2direct.ncu-rep --hot 30 > gpurun_out/ncu_direct_summary.txt 2>&1; head -20 gpurun_out/ncu_direct_summary.txt
