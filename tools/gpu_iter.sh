# build-measure loop on the GPU box: parity tests, a short bench, one ncu capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
LSK_CPU_ITERS=2 timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
for n in 148 1184 8192; do python tools/profile_dense.py --n $n --iters 200 --reps 3; done > gpurun_out/prof_plain.log 2>&1
if [ "${LSK_NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_solve_dense -c 1 -o gpurun_out/dense_k100 -f python tools/profile_dense.py --iters 100 > gpurun_out/ncu1.log 2>&1
fi
cat gpurun_out/pytest_gpu.log gpurun_out/prof_plain.log; tail -2 gpurun_out/bench.log
