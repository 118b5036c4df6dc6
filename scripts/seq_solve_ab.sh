set -x
O=gpurun_out
timeout 900 python -m pytest tests/test_refldl_gpu.py -x -q > $O/seq_refldl_tests.txt 2>&1
for v in 1 0; do
  OCG_REFLDL_SOLVE=$v timeout 300 python scripts/refldl_bench.py goddard:1000 goddard:2000 quadrotor:2000 >> $O/seq_refldl_bench_$v.jsonl 2>&1
  OCG_REFLDL_SOLVE=$v timeout 600 python scripts/goddard_parity.py 1000 >> $O/seq_goddard_parity_$v.jsonl 2>&1
done
