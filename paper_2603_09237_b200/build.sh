#!/usr/bin/env bash
# Builds libmorlax_b200.so in-tree for sm_100a (B200). Used by build() in
# __graft_entry__.py and by the Python loader when the .so is missing.
set -euo pipefail
cd "$(dirname "$0")"
NVCC=${NVCC:-nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="-O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr -Xptxas -v"
mkdir -p build
SRCS="csrc/kernels.cu csrc/pareto.cu csrc/trainer.cu csrc/comm.cu csrc/capi.cu csrc/rollout_tc.cu csrc/img_gemm.cu csrc/feature.cu csrc/hv_exact.cu csrc/policy.cu csrc/evaluate.cu csrc/dm_adam.cu"
pids=()
objs=()
for s in $SRCS; do
  o=build/$(basename "$s" .cu).o
  objs+=("$o")
  ( $NVCC $ARCH $FLAGS -c "$s" -o "$o" > "build/$(basename "$s" .cu).log" 2>&1 || { cat "build/$(basename "$s" .cu).log"; exit 1; } ) &
  pids+=($!)
done
rc=0
for p in "${pids[@]}"; do wait "$p" || rc=1; done
[ $rc -eq 0 ] || exit 1
$NVCC $ARCH -shared -o libmorlax_b200.so "${objs[@]}" -ldl
echo "built $(pwd)/libmorlax_b200.so"
