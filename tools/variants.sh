#!/usr/bin/env bash
# Build A/B variants of the library for one GPU session:
#   tools/variants.sh NAME "DEFINES" [NAME "DEFINES" ...]
# -> variants/libec3r_NAME.so; select one with EC3R_B200_LIB=variants/libec3r_NAME.so
set -eu
make -s
mkdir -p variants build/var
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude"
while [ $# -ge 2 ]; do
    name=$1; defs=$2; shift 2
    objs=""
    for src in paper_2510_02080_b200/csrc/*.cu; do
        b=$(basename "$src" .cu)
        o=build/var/${name}_$b.o
        nvcc $NVFLAGS $defs -dc -c "$src" -o "$o"
        objs="$objs $o"
    done
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libec3r_$name.so $objs -lcudart_static -lrt -ldl -lpthread
    echo "built variants/libec3r_$name.so ($defs)"
done
