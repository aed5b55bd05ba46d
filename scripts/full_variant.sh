# usage: bash scripts/full_variant.sh NAME "-DFOO=1 ..." -> paper_1711_01228_b200/lib_ab/libfdl_NAME.so
# (all three sources rebuilt with the definitions; scratch_variants.sh rebuilds fdl_sym.cu only)
set -e
NAME=$1; DEFS=$2; D=/tmp/fvar_$NAME; mkdir -p $D paper_1711_01228_b200/lib_ab
for f in fdl_sym fdl_kernels fdl_api; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O2 \
    --expt-relaxed-constexpr -diag-suppress 128 $DEFS -I include -c paper_1711_01228_b200/csrc/$f.cu -o $D/$f.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1711_01228_b200/lib_ab/libfdl_$NAME.so \
  $D/fdl_sym.o $D/fdl_kernels.o $D/fdl_api.o -cudart shared -ldl -Xlinker --no-undefined
echo built lib_ab/libfdl_$NAME.so
