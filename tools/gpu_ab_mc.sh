export LSK_AB="paper_2605_00837_b200/liblsk.so build/liblsk_counter.so"
export LSK_AB_ARGS="--n_8192_--eps_1e-3 --n_148_--m_8192_--eps_1e-3 --n_1024_--eps_1e-2 --n_1024_--eps_1e-2_--no-cluster --n_4096_--m_1024_--eps_1e-2"
bash tools/gpu_ab.sh
bash tools/gpu_ab.sh > /dev/null; cat gpurun_out/ab.log
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
