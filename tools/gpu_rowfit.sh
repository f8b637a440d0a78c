# per-row time and per-iteration overhead of the dense kernels (m = 8192; linear fit over n)
mkdir -p gpurun_out
for n in 1184 2368 4736 8192; do for t in "" "--one-team"; do echo "n=$n $t $(timeout 120 python tools/profile_dense.py --n $n --m 8192 --iters 200 --reps 3 $t 2>&1 | tail -1)"; done; done > gpurun_out/rowfit.log 2>&1
cat gpurun_out/rowfit.log
