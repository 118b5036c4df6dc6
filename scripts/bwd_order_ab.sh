#!/bin/bash
# reference-order solve with the backward terms subtracted in entry order:
# the refldl GPU tests (Goddard@1000 = 510, @2500 = 1737 iterations), the
# per-solve time and the Goddard@1000 parity solve against the reference
O=gpurun_out
timeout 1200 python -m pytest tests/test_refldl_gpu.py tests/test_ipm_gpu.py -x -q > $O/bwd_tests.txt 2>&1
timeout 300 python scripts/refldl_bench.py goddard:1000 goddard:2000 > $O/bwd_refldl_bench.jsonl 2>&1
timeout 600 python scripts/goddard_parity.py 1000 > $O/bwd_goddard_parity.jsonl 2>&1
