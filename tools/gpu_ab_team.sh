# A/B of ablation builds of the dense kernels (timing only; ablations compute wrong results)
mkdir -p gpurun_out
for lib in paper_2605_00837_b200/liblsk.so build/liblsk_pf2.so build/liblsk_pf3.so build/liblsk_pf5.so build/liblsk_t_NOWAIT.so build/liblsk_t_NOMUFU.so build/liblsk_t_NOBAR.so build/liblsk_t_NOFIN.so; do
  for n in 1184 8192; do
    echo "$lib n=$n $(LSK_LIB=$lib timeout 120 python tools/profile_dense.py --n $n --m 8192 --iters 200 --reps 3 2>&1 | tail -1)"
  done
done > gpurun_out/ab_team.log 2>&1
echo "one-team n=8192 $(timeout 120 python tools/profile_dense.py --n 8192 --iters 200 --reps 3 --one-team 2>&1 | tail -1)" >> gpurun_out/ab_team.log
cat gpurun_out/ab_team.log
