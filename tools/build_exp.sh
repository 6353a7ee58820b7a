#!/bin/bash
# Build an experiment variant of the library: tools/build_exp.sh NAME -DMACRO ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=paper_2408_02350_b200/build/exp_$name
mkdir -p $out
rm -f $out/*.o $out/*.so
pids=()
for f in paper_2408_02350_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" -c $f -o $out/$(basename $f).o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p || { echo "build failed" >&2; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libbgk_b200.so $out/*.o
echo $out/libbgk_b200.so
