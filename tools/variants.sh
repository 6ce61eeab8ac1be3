#!/bin/bash
# Build libgfq variants into paper_2507_08954_b200/var_*.so: name then extra nvcc flags.
set -e
cd "$(dirname "$0")/.."
build() { n=$1; shift; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 "$@" -Xcompiler -fPIC -shared -Iinclude -o paper_2507_08954_b200/var_$n.so paper_2507_08954_b200/csrc/gfq_engine.cu; }
build O2 -Xptxas -O2 & build O1 -Xptxas -O1 & build m5 -DGFQ_MINB=5 & build m6 -DGFQ_MINB=6 & wait
for f in paper_2507_08954_b200/var_*.so; do echo "$f $(cuobjdump -sass $f | awk '/Function :/{name=$3} /^        \/\*[0-9a-f]+\*\//{c[name]++} END{print c["_ZN3gfq5k_simILb0EEEvNS_6ParamsE"]}')"; done
