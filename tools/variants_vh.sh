#!/usr/bin/env bash
# Fast A/B variants of the fusion kernels only: recompiles vhash.cu with the
# given defines (in parallel) and links it with the other objects of `make`.
#   tools/variants_vh.sh NAME "DEFINES" [NAME "DEFINES" ...]
# -> variants/libec3r_NAME.so; select one with EC3R_B200_LIB=variants/libec3r_NAME.so
set -eu
make -s
mkdir -p variants build/var
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude"
others=$(ls build/*.o | grep -v '/vhash.o$')
pids=""
while [ $# -ge 2 ]; do
    name=$1; defs=$2; shift 2
    (
        nvcc $NVFLAGS $defs -dc -c paper_2510_02080_b200/csrc/vhash.cu -o build/var/${name}_vhash.o 2>/dev/null
        nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libec3r_$name.so build/var/${name}_vhash.o $others \
            -lcudart_static -lrt -ldl -lpthread
        echo "built variants/libec3r_$name.so ($defs)"
    ) &
    pids="$pids $!"
done
for p in $pids; do wait $p; done
