#!/bin/bash
# Build an experimental variant of the library: tools/build_variant.sh NAME "-DFLAG=V ..."
# -> paper_2005_09904_b200/lib/libbiqgemm_b200.NAME.so (select with BQG_LIB_VARIANT=NAME)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/var_$name; mkdir -p $out paper_2005_09904_b200/lib
for f in paper_2005_09904_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I include $@ -c $f -o $out/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2005_09904_b200/lib/libbiqgemm_b200.$name.so $out/*.o -lcudart_static -lrt -ldl -lpthread
