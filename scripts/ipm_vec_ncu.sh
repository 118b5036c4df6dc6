#!/bin/bash
# ncu (no replay of the whole app: per-kernel metrics) of the device IPM's
# vector kernels (csrc/ipm_kernels.cu, namespace ipmdev) during a quadrotor
# N=1e5 solve: duration and DRAM bytes per launch, first 60 launches.
O=${1:-gpurun_out/ipm_vec_ncu.csv}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size \
  --clock-control none -k "regex:^(accept_k|barrier_k|dphi_k|dual_dir_k|expand_k|finalize_k|ftb_k|kkt_error_k|l1_k|resid_k|residual_k|rhs_k|sigma_k|trial_scatter_dev_k|sym_matvec_k|jt_lambda_k|kkt_assemble_tiled_k)$" -c 80 --csv --log-file $O \
  python -c "
import sys; sys.path.insert(0, '.')
from paper_2510_03932_b200 import MODELS, Model, solve
r = solve(Model(MODELS['quadrotor'], 100000))
print(r['iterations'], r['objective'])
" > ${O%.csv}.log 2>&1
