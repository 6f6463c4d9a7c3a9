#!/bin/bash
# Dev tool: libpentab.so variants with extra -D flags on chosen sources.
# usage: tools/build_variants2.sh name "src1.cu src2.cu" "-DFOO=1 ..."
set -e
cd "$(dirname "$0")/.."
CS=paper_2101_06550_b200/csrc
B=paper_2101_06550_b200/build
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -cudart static -I include"
name=$1; srcs=$2; D=$3
mkdir -p /tmp/var_$name tools/variants
objs=$(ls $B/*.o)
for s in $srcs; do
  o=${s%.cu}.o
  nvcc $FL $D -c $CS/$s -o /tmp/var_$name/$o
  objs=$(echo "$objs" | grep -v "/$o\$")
  objs="$objs /tmp/var_$name/$o"
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/variants/v_$name.so $objs
echo built $name
