# one ncu --set full capture of the dense kernel at C2 (40 iterations): NAME=<tag> EXTRA="<profile_dense args>"
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_solve_dense -c 1 -o gpurun_out/dense_${NAME:-x} -f python tools/profile_dense.py --iters 40 $EXTRA > gpurun_out/ncu_${NAME:-x}.log 2>&1; echo "ncu rc $?"
