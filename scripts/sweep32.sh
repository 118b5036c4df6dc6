#!/bin/bash
# one-warp-block sweep of the fused J+H kernel at Goddard N=1e5: register
# budget (min resident blocks), output staging (split), input staging
O=${1:-gpurun_out/sweep32.jsonl}
timeout 1500 python scripts/sweep_eval.py goddard:100000 quadrotor:100000 --block 32 --minb 0,16,18,20,22 --split=-1,0,1 --staging=-1,0 --steps 30 >> $O 2> ${O%.jsonl}.err
