# A/B of library builds on the dense profile: LSK_AB="lib1 lib2 ..." LSK_AB_ARGS="--n 8192 ..." 
mkdir -p gpurun_out
for lib in ${LSK_AB}; do
  for args in ${LSK_AB_ARGS:-"--n 8192"}; do
    a=${args//_/ }
    echo "$lib [$a] $(LSK_LIB=$lib timeout 120 python tools/profile_dense.py $a --iters 200 --reps 3 2>&1 | tail -1)"
  done
done > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
