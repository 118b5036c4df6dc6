#!/bin/bash
# A/B of the drop-in's staging copies (integration/xfer.hpp):
# OCTRANS_ACCEL_XFER = chunk_doubles,slots,threads,nt (nt bit 0: streaming
# stores into the caller's vectors on D2H, bit 1: into the staging slots on H2D)
O=${1:-gpurun_out/dropin_nt_ab.txt}
for rep in 1 2; do
for cfg in 262144,6,8,0 262144,6,8,1 262144,6,8,3 262144,6,12,1 524288,4,8,1 131072,8,8,1 262144,6,6,1; do
  echo "cfg $cfg $(OCTRANS_ACCEL_XFER=$cfg timeout 300 python scripts/dropin_e2e.py goddard:100000 2>&1 | tail -1)" >> $O
done
done
