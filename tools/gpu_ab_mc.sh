export LSK_AB="paper_2605_00837_b200/liblsk.so build/liblsk_chkdirect.so"
export LSK_AB_ARGS="--n_8192_--eps_1e-3 --n_8192_--eps_1e-3_--check_1000 --n_4096_--m_8192_--eps_1e-3"
bash tools/gpu_ab.sh
