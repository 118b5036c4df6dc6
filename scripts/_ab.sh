O=gpurun_out
T=r2_kt1
timeout 900 python -m pytest tests/test_kkt_gpu.py tests/test_ipm_gpu.py -m gpu -x -q > $O/${T}_tests.txt 2>&1
timeout 600 python scripts/kkt_roofline.py goddard:100000 quadrotor:100000 > $O/${T}_roof.jsonl 2> $O/${T}_roof.err
OCG_KKT_TILED=0 timeout 600 python scripts/kkt_roofline.py goddard:100000 quadrotor:100000 > $O/${T}_roof_untiled.jsonl 2>> $O/${T}_roof.err
timeout 600 ncu --set full --clock-control none -k regex:kkt_assemble -c 2 -o $O/${T}_prof -f python scripts/kkt_roofline.py goddard:100000 > /dev/null 2>> $O/${T}_roof.err
