# end-of-round check: tests, smoke, bench + launch list, one ncu capture of the dense kernel, sanitizers
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $? $(tail -1 gpurun_out/pytest_gpu.log)"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; cat gpurun_out/smoke.log | tail -4
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc $?"; tail -1 gpurun_out/bench_full.log > gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > gpurun_out/bench_ncu.log 2>&1; echo "ncu rc $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_solve_dense -c 1 -o gpurun_out/dense_r2final -f python tools/profile_dense.py --iters 40 > gpurun_out/ncu_final.log 2>&1; echo "ncu full rc $?"
for tool in memcheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc $? $(grep 'SUMMARY' gpurun_out/san_$tool.log)"
done
LSK_LIB=build/liblsk_san.so timeout 900 compute-sanitizer --tool racecheck --print-limit 30 python tools/sanitize.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc $? $(grep 'SUMMARY' gpurun_out/san_racecheck.log)"
