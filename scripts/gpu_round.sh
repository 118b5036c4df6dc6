#!/bin/bash
# One gpurun call: GPU parity tests, bench lines, ncu launch list + full capture.
# usage: scripts/gpu_round.sh TAG   (outputs under gpurun_out/TAG_*)
T=${1:-r2}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${T}_env.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $O/${T}_gputests.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.txt 2>&1
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/${T}_bench_ref.json 2>> $O/${T}_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary --solve none --goddard-solve none --goddard-parity none --batch none > /dev/null 2>> $O/${T}_ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ocg_cjh -s 1 -c 1 -o $O/${T}_prof_goddard -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary --solve none --goddard-solve none --goddard-parity none --batch none > /dev/null 2>> $O/${T}_ncu.err
timeout 900 bash scripts/ipm_vec_ncu.sh $O/${T}_ipm_vec_ncu.csv
echo done
