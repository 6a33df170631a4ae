#!/bin/bash
# ncu captures of the NEXT-mode kernels (run under gpurun, 1 GPU).  Usage: tools/profile_next.sh <tag>
# tools/next_modes.py launches, in order: grid encode + U-Net, query_cells (select, head<0,1>),
# query_grad (crop path, head_tc<1,1>), closed loop (sim_prepare, select, head_tc<0,1>, sim_integrate, ...).
# The context is bf16, so the predictor is the tensor-core kernel (head_tc_kernel<kProj, kGrad>).
TAG=${1:-r1next}
mkdir -p gpurun_out
python tools/next_modes.py > gpurun_out/next_plain_$TAG.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/next_launches_$TAG.csv \
    python tools/next_modes.py > /dev/null 2>&1
cap() {  # name regex skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o gpurun_out/next_${TAG}_$1 \
      python tools/next_modes.py > gpurun_out/ncu_next_${TAG}_$1.log 2>&1 || true
  ncu -i gpurun_out/next_${TAG}_$1.ncu-rep --page details > gpurun_out/next_details_${TAG}_$1.txt 2>/dev/null || true
  ncu -i gpurun_out/next_${TAG}_$1.ncu-rep --page raw --csv > gpurun_out/next_raw_${TAG}_$1.csv 2>/dev/null || true
}
# bf16 context: the grid encode is 4 conv_tc (ntaps = 1) GEMMs (layer 1 fused) -> cell_max per chunk of shapes
# (2 chunks at 1030 x 1500 points), so the U-Net's c1 is the 9th conv_tc launch and d1 the 16th
cap grid_gemm conv_tc 0
cap grid_cellmax cell_max 0
cap conv_c1 conv_tc 8
cap conv_d1 conv_tc 15
cap cells_select cells_select 0
cap head_cells head_tc 0
cap head_grad head_tc 1
cap sim_integrate sim_integrate 0
