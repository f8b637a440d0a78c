mkdir -p gpurun_out
{ nproc; lscpu | grep -i "model name\|numa\|socket\|MHz" ; 
for kb in 1024 4096 16384; do echo "== chunk ${kb} KB"; LSK_H2D_CHUNK_KB=$kb PROBE_T="0 8 16" timeout 300 python tools/h2d_probe.py; done; } > gpurun_out/h2d.log 2>&1
cat gpurun_out/h2d.log
