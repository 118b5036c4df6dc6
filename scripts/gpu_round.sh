#!/bin/bash
# One gpurun call: GPU parity tests, bench lines, ncu launch list + full capture.
# usage: scripts/gpu_round.sh TAG   (outputs under gpurun_out/TAG_*)
T=${1:-r1}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${T}_env.txt
timeout 1200 python -m pytest tests -m gpu -q > $O/${T}_gputests.txt 2>&1
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $O/${T}_bench_ref.json 2>> $O/${T}_bench.err
timeout 300 python bench.py --no-cpu-baseline --solve none --goddard-solve none --batch none --secondary > $O/${T}_bench_secondary.json 2>> $O/${T}_bench.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 10 --warmup 3 --solve none --goddard-solve none --batch none > $O/${T}_bench_2rank.json 2>> $O/${T}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 3 --warmup 1 --no-cpu-baseline --solve none --goddard-solve none --batch none > /dev/null 2>> $O/${T}_ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ocg_cjh -s 1 -c 1 -o $O/${T}_prof_goddard -f \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --solve none --goddard-solve none --batch none > /dev/null 2>> $O/${T}_ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ocg_cjh -s 1 -c 1 -o $O/${T}_prof_quad1e6 -f \
  python bench.py --model quadrotor --N 1000000 --steps 1 --warmup 1 --no-cpu-baseline --solve none --goddard-solve none --batch none > /dev/null 2>> $O/${T}_ncu.err
echo done
