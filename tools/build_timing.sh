#!/bin/bash
# Debug build with clock64 phase counters (OFDMR_PHASE_TIMING) -> libofdmr_b200_timing.so
set -e
cd "$(dirname "$0")/../paper_2209_03883_b200"
mkdir -p _build_t
F="-O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -DOFDMR_PHASE_TIMING"
objs=""
for u in radar_kernels mixed_kernels colpass2048 fast_kernels fused_ce fused_pg2 fused_pg3 rowpass_zp noise_kernels ofdm_kernels io_kernels capi multi sft_kernels gen_kernels; do
  ex=""; case $u in sft_kernels|gen_kernels) ex="-fmad=false";; esac
  nvcc $F $ex -c csrc/$u.cu -o _build_t/$u.o & objs="$objs _build_t/$u.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libofdmr_b200_timing.so $objs -lcudart
