#!/usr/bin/env bash
# Fast A/B variants of one source file: recompiles it (vhash.cu unless
# EC3R_VAR_SRC names another csrc file) with the given defines, in parallel,
# and links it with the other objects of `make`.
#   [EC3R_VAR_SRC=umeyama] tools/variants_vh.sh NAME "DEFINES" [NAME "DEFINES" ...]
# -> variants/libec3r_NAME.so; select one with EC3R_B200_LIB=variants/libec3r_NAME.so
set -eu
make -s
mkdir -p variants build/var
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude"
SRC=${EC3R_VAR_SRC:-vhash}
others=$(ls build/*.o | grep -v "/$SRC.o\$")
pids=""
while [ $# -ge 2 ]; do
    name=$1; defs=$2; shift 2
    (
        nvcc $NVFLAGS $defs -dc -c paper_2510_02080_b200/csrc/$SRC.cu -o build/var/${name}_$SRC.o 2>/dev/null
        nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libec3r_$name.so build/var/${name}_$SRC.o $others \
            -lcudart_static -lrt -ldl -lpthread
        echo "built variants/libec3r_$name.so ($defs)"
    ) &
    pids="$pids $!"
done
for p in $pids; do wait $p; done
