#!/bin/bash
T=${1:-sweep}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/${T}_gputests.txt 2>&1
timeout 900 python scripts/sweep_eval.py --minb 0 --split 0,2 > $O/${T}_sweep.jsonl 2> $O/${T}_sweep.err
timeout 600 python bench.py --no-cpu-baseline > $O/${T}_bench.json 2> $O/${T}_bench.err
echo done
