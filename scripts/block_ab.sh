#!/bin/bash
# bench headline (Goddard N=1e5 fused J+H, 50 event-timed steps) with one-warp
# vs four-warp blocks, alternated
O=${1:-gpurun_out/block_ab.jsonl}
for rep in 1 2 3; do
  for b in 32 128; do
    timeout 300 python bench.py --block $b --steps 50 --no-cpu-baseline --no-secondary --solve none --goddard-solve none \
      --goddard-parity none --batch none 2>/dev/null | tail -1 | python -c "
import json,sys; o=json.loads(sys.stdin.read()); print(json.dumps({'block': $b, 'rep': $rep, 'us': o['ms_per_step']*1e3, 'frac': o['roofline']['frac'], 'e2e_c_abi': o.get('e2e_c_abi',{}).get('value')}))" >> $O
  done
done
