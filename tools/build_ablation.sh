# build/liblsk_<name>.so: the library with lsk_api.cu compiled under extra -D flags (timing ablations only)
# usage: bash tools/build_ablation.sh name -DLSK_X_NOWAIT ...   (UNIT=lsk_points.cu: flags on that unit instead)
set -e
name=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null
INC=$(python -c "import paper_2605_00837_b200._build as b; print(b.nccl_dirs()[0])")
LIBD=$(python -c "import paper_2605_00837_b200._build as b; print(b.nccl_dirs()[1])")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC -I$INC "$@" \
  -c paper_2605_00837_b200/csrc/${UNIT:-lsk_api.cu} -o build/abl_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/liblsk_$name.so build/abl_$name.o \
  $(python -c "import paper_2605_00837_b200._build as b; print(' '.join('build/' + u.replace('.cu', '.o') for u in b.UNITS if u != '${UNIT:-lsk_api.cu}'))") -lcuda -Xlinker $LIBD/libnccl.so.2 -Xlinker -rpath=$LIBD
