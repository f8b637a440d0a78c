export LSK_AB="paper_2605_00837_b200/liblsk.so"
export LSK_AB_ARGS="--n_8192_--eps_1e-3 --n_8192_--eps_1e-3_--direct --n_8192_--eps_1e-3_--direct_--check_1000 --n_8192_--eps_1e-3_--direct_--general --n_8192_--eps_1e-4"
bash tools/gpu_ab.sh
