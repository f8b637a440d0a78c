for a in "--n 1024 --eps 1e-2" "--n 1024 --eps 1e-2 --direct" "--n 1024 --eps 1e-2 --no-cluster" "--n 1024 --eps 1e-2 --no-cluster --direct" "--n 512 --m 1024 --eps 1e-2 --direct" "--n 128 --m 1024 --eps 1e-2 --direct"; do
  echo "[$a] $(timeout 120 python tools/profile_dense.py $a --iters 200 --reps 3 2>&1 | tail -1)"
done
