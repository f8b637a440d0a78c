export LSK_AB="paper_2605_00837_b200/liblsk.so build/liblsk_mc4.so"
export LSK_AB_ARGS="--n_256_--m_1024_--eps_1e-2 --n_512_--m_1024_--eps_1e-2 --n_1024_--eps_1e-2 --n_2048_--m_1024_--eps_1e-2 --n_4096_--m_1024_--eps_1e-2"
bash tools/gpu_ab.sh
LSK_VERBOSE=1 LSK_LIB=$PWD/build/liblsk_mc4.so python tools/solver_selection_probe.py 2>&1 | tail -8
LSK_LIB=$PWD/build/liblsk_mc4.so timeout 900 python -m pytest tests/test_gpu_cluster.py -q -x -p no:cacheprovider 2>&1 | tail -2
