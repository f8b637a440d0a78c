# build/liblsk_san.so: every unit compiled with -DLSK_X_ALLARRIVE (every thread
# arrives on the row-sum mbarriers) for compute-sanitizer racecheck runs:
#   LSK_LIB=build/liblsk_san.so compute-sanitizer --tool racecheck python tools/sanitize.py
set -e
python - <<'PY'
import os, subprocess
import paper_2605_00837_b200._build as b
inc, libdir = b.nccl_dirs()
os.makedirs("build/san", exist_ok=True)
objs = []
for u in b.UNITS:
    o = "build/san/" + u.replace(".cu", ".o")
    subprocess.run([b.nvcc(), *b.ARCH, *b.FLAGS, "-DLSK_X_ALLARRIVE", "-I" + inc, "-c", os.path.join(b.CSRC, u), "-o", o], check=True)
    objs.append(o)
subprocess.run([b.nvcc(), *b.ARCH, "-shared", "-o", "build/liblsk_san.so", *objs, "-lcuda", "-Xlinker",
                os.path.join(libdir, "libnccl.so.2"), "-Xlinker", "-rpath=" + libdir], check=True)
print("build/liblsk_san.so")
PY
