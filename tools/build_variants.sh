#!/bin/bash
# Dev tool: build libpentab.so variants with different two-pass ring shapes
# (TP_NC*/TP_R* of fused_part.cuh) into tools/variants/ for a GPU sweep.
# usage: tools/build_variants.sh name "NC1 R1 NC2 R2" [name "..."] ...
set -e
cd "$(dirname "$0")/.."
CS=paper_2101_06550_b200/csrc
B=paper_2101_06550_b200/build
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -cudart static -I include"
while [ $# -ge 2 ]; do
  name=$1; set -- $2 "${@:3}"; a=$1; b=$2; c=$3; d=$4; shift 4
  D="$EXTRA -DTP_NC1_64=$a -DTP_R1_64=$b -DTP_NC2_64=$c -DTP_R2_64=$d -DTP_NC1_32=4 -DTP_R1_32=4 -DTP_NC2_32=4 -DTP_R2_32=4"
  mkdir -p /tmp/var_$name
  nvcc $FL $D -c $CS/fused_part_f64_inter.cu -o /tmp/var_$name/f64.o &
  nvcc $FL $D -c $CS/fused_part_f32_inter.cu -o /tmp/var_$name/f32.o &
  wait
  objs=$(ls $B/*.o | grep -v fused_part_f64_inter | grep -v fused_part_f32_inter)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o tools/variants/v_$name.so $objs /tmp/var_$name/f64.o /tmp/var_$name/f32.o
  echo built $name
done
