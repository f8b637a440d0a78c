# A/B of two library builds on the dense profile (m = 8192 fixed, n varies: L2-resident vs HBM)
mkdir -p gpurun_out
for lib in ${LSK_AB:-paper_2605_00837_b200/liblsk.so}; do  # LSK_AB="a.so b.so": libraries to compare
  for nm in "148 8192" "1184 8192" "2368 8192" "8192 8192"; do
    set -- $nm
    echo "$lib n=$1 m=$2 $(LSK_LIB=$PWD/$lib python tools/profile_dense.py --n $1 --m $2 --iters 200 --reps 3)"
  done
done > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
