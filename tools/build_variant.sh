#!/bin/bash
# Build an A/B variant of libsbnet.so with extra nvcc flags into tools/bin/<name>.so
# (then: SBN_LIB_PATH=tools/bin/<name>.so python tools/...):
#   tools/build_variant.sh ns64 -DSBN_FWAIT_NS=64
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=/tmp/sbn_variant_$name
mkdir -p "$root/tools/bin"
mkdir -p "$out"
objs=()
for f in "$root"/paper_1801_02108_b200/csrc/*.cu; do
  o=$out/$(basename "${f%.cu}").o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I"$root/include" "$@" -c "$f" -o "$o" 2>/dev/null &
  objs+=("$o")
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/tools/bin/$name.so" "${objs[@]}" -lcuda
echo "$root/tools/bin/$name.so"
