timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_sharded.py tests/test_gpu_points.py tests/test_gpu_fuzz_points.py -q -p no:cacheprovider 2>&1 | tail -6
timeout 900 python tools/profile_sharded.py > gpurun_out/sharded.md 2>&1; cat gpurun_out/sharded.md
