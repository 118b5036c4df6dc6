#!/bin/bash
# usage: scripts/gpu_prof.sh TAG  — ncu full captures of the fused kernel + solve bench
T=${1:-prof}
O=gpurun_out
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ocg_cjh -s 1 -c 1 -o $O/${T}_prof_goddard -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>> $O/${T}_ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ocg_cjh -s 1 -c 1 -o $O/${T}_prof_quad1e6 -f \
  python bench.py --model quadrotor --N 1000000 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>> $O/${T}_ncu.err
timeout 1500 python scripts/solve_bench.py double_integrator:100000 quadrotor:2000 goddard:1000 quadrotor:20000 > $O/${T}_solves.jsonl 2> $O/${T}_solves.err
echo done
