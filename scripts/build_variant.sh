#!/bin/bash
# Experimental build of libsgmv_b200.so with extra nvcc flags into build/variants/<name>/.
# To measure it, copy it over paper_2310_18547_b200/lib/libsgmv_b200.so inside the gpurun command
# (the product loader has no override hook).
# Usage: scripts/build_variant.sh <name> <extra nvcc flags...>
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/build/variants/$name
mkdir -p $out
flags="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I$root/include $*"
pids=()
for f in $root/paper_2310_18547_b200/csrc/*.cu; do
  nvcc $flags -c $f -o $out/$(basename $f).o & pids+=($!)
done
for p in ${pids[@]}; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libsgmv_b200.so $out/*.o
rm -f $out/*.o  # only the library travels to the GPU box
echo built $out/libsgmv_b200.so
