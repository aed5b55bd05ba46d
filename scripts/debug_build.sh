# usage: bash scripts/debug_build.sh  -> paper_1711_01228_b200/lib_ab/libfdl_dbg.so
# The library with FDL_DEBUG_BOUNDS: kernels check their global-memory indices and trap on a
# violation (compute-sanitizer is closed on this GPU pool).  Run the GPU tests against it with
#   FDL_LIB=$PWD/paper_1711_01228_b200/lib_ab/libfdl_dbg.so python -m pytest tests -m gpu
set -e
D=/tmp/fdl_dbg; mkdir -p $D paper_1711_01228_b200/lib_ab
for f in fdl_sym fdl_kernels fdl_api; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O2 \
    --expt-relaxed-constexpr -diag-suppress 128 -DFDL_DEBUG_BOUNDS -I include \
    -c paper_1711_01228_b200/csrc/$f.cu -o $D/$f.o
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1711_01228_b200/lib_ab/libfdl_dbg.so \
  $D/fdl_sym.o $D/fdl_kernels.o $D/fdl_api.o -cudart shared -ldl -Xlinker --no-undefined
echo built paper_1711_01228_b200/lib_ab/libfdl_dbg.so
