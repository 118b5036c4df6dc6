#!/bin/bash
# usage: scripts/gpu_sweep.sh TAG MINB_LIST [pytest-args]
T=${1:-sweep}
MB=${2:-0}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q ${3:-} > $O/${T}_gputests.txt 2>&1
timeout 1500 python scripts/sweep_eval.py --minb $MB --split ${4:--1} ${5:-} > $O/${T}_sweep.jsonl 2> $O/${T}_sweep.err
echo done
