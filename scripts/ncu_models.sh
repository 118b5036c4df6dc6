#!/bin/bash
# ncu --set full of the fused J+H kernel for the other N=1e5 eval configs
# (one capture each, as bench.py launches the headline: L2 flushed before)
O=${1:-gpurun_out}
for m in hang_glider shuttle quadrotor; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:ocg_cjh -s 1 -c 1 -o $O/r2_ncu_${m}_cjh -f \
    python bench.py --model $m --steps 1 --warmup 3 --no-cpu-baseline --no-secondary --solve none --goddard-solve none \
      --goddard-parity none --batch none > /dev/null 2>> $O/ncu_models.err
done
