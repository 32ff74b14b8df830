#!/bin/bash
# Build libtk_sm100.so variants with compile-time knobs into build/var_<name>/ (tuning only).
# usage: tools/build_variants.sh name1 "-DFOO=1 -DBAR=2" name2 "-D..." ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
pids=()
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p "$ROOT/build/var_$name"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
    -cudart static $flags -o "$ROOT/build/var_$name/libtk_sm100.so" "$ROOT/paper_2009_12263_b200/csrc/tk_api.cu" \
    > "$ROOT/build/var_$name/build.log" 2>&1 &
  pids+=($!)
done
rc=0
for p in "${pids[@]}"; do wait $p || rc=1; done
exit $rc
