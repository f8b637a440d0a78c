# host -> device staging of C2's fp64 matrix: chunk size x non-temporal stores x worker threads
mkdir -p gpurun_out
{ nproc; lscpu | grep -i "model name\|numa\|socket\|L3"
for nt in 1 0; do for kb in 512 1024 2048; do echo "== NT ${nt} chunk ${kb} KB"; LSK_H2D_NT=$nt LSK_H2D_CHUNK_KB=$kb PROBE_T="${PROBE_T:-0 8 16}" timeout 300 python tools/h2d_probe.py; done; done; } > gpurun_out/h2d.log 2>&1
cat gpurun_out/h2d.log
