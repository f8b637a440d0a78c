# compute-sanitizer (all four tools) over the cluster dense solvers only (tools/sanitize.py cluster)
export LSK_VERBOSE=1
mkdir -p gpurun_out
python tools/sanitize.py cluster > gpurun_out/san_cluster_plain.log 2>&1; echo "plain rc $?"; tail -3 gpurun_out/san_cluster_plain.log
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py cluster > gpurun_out/san_cluster_$tool.log 2>&1; echo "$tool rc $? $(grep 'SUMMARY' gpurun_out/san_cluster_$tool.log)"
done
for tool in memcheck racecheck; do echo "$tool: $(grep -c 'clusters of' gpurun_out/san_cluster_$tool.log) multi-cluster launches, $(grep -c 'single cluster' gpurun_out/san_cluster_$tool.log) single, $(grep -c 'grid of' gpurun_out/san_cluster_$tool.log) grid"; done
timeout 600 python -m pytest tests/test_gpu_cluster.py -q -p no:cacheprovider 2>&1 | tail -2
