mkdir -p gpurun_out
LSK_LIB=build/liblsk_allarrive.so timeout 900 compute-sanitizer --tool racecheck --print-limit 30 python tools/sanitize.py > gpurun_out/sanitize_racecheck_allarrive.log 2>&1; echo "racecheck rc $?"
tail -3 gpurun_out/sanitize_racecheck_allarrive.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_solve_dense -c 1 -o gpurun_out/dense_r2a -f python tools/profile_dense.py --iters 40 > gpurun_out/ncu_r2a.log 2>&1; echo "ncu rc $?"
echo done
