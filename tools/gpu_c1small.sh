for a in "--n 16 --m 1024 --eps 1e-2" "--n 128 --m 1024 --eps 1e-2" "--n 128 --m 1024 --eps 1e-2 --no-cluster"; do
  echo "[$a] $(timeout 120 python tools/profile_dense.py $a --iters 200 --reps 3 2>&1 | tail -1)"
done
NAME=c1c EXTRA="--n 128 --m 1024 --eps 1e-2" bash tools/gpu_ncu_dense.sh
