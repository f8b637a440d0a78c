export LSK_AB="paper_2605_00837_b200/liblsk.so build/liblsk_bcast.so"
export LSK_AB_ARGS="--n_256_--m_1024_--eps_1e-2 --n_512_--m_1024_--eps_1e-2 --n_1024_--eps_1e-2 --n_2048_--m_1024_--eps_1e-2 --n_4096_--m_1024_--eps_1e-2"
bash tools/gpu_ab.sh
bash tools/gpu_ab.sh > /dev/null; cat gpurun_out/ab.log
LSK_LIB=$PWD/build/liblsk_trace.so python tools/trace_cluster.py 1024 1024 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
