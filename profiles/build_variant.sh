# build an alternate libgvx_cuda.so with extra nvcc defines into variants/<name>/
# usage: bash profiles/build_variant.sh <name> "<-DFOO=1 ...>"
set -e
NAME=$1; DEFS=$2
ARCH="-gencode arch=compute_100a,code=sm_100a"
mkdir -p variants/$NAME/obj
for f in paper_2008_11476_b200/csrc/cuda/*.cu; do
  b=$(basename $f .cu)
  nvcc $ARCH -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2008_11476_b200/csrc/cuda $DEFS -Xptxas -v -c $f -o variants/$NAME/obj/$b.o 2> variants/$NAME/obj/$b.log &
done
wait
nvcc $ARCH -shared -Xcompiler -fPIC variants/$NAME/obj/*.o -o variants/$NAME/libgvx_cuda.so -L/usr/local/cuda/lib64 -lnvrtc -Xlinker -rpath,/usr/local/cuda/lib64
grep -h -A2 "harris_kernel\|edge_kernel\|sep_kernel" variants/$NAME/obj/*.log | grep -E "registers|spill" | sort | uniq -c | head -5
