# round-2: lane fp16 fast path
cd $GRAFT_REPO_ROOT
( FG_VQ_LANE=2 timeout 900 python -m pytest tests/test_gpu_aggregate.py -x -q -k vq ) > gpurun_out/t_l.log 2>&1
( timeout 900 python -m pytest tests/test_gpu_aggregate.py -x -q -k vq ) >> gpurun_out/t_l.log 2>&1
grep -E "passed|failed" gpurun_out/t_l.log
timeout 900 python tools/fused_bench.py --config mag240m --iters 20 --check 2>&1 | grep -E "avg_us|check"
FG_VQ_LANE=2 timeout 900 python tools/fused_bench.py --config products --iters 20 --check 2>&1 | grep -E "avg_us|check"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_vq_mean8" --launch-skip 3 -c 1 \
   -o gpurun_out/mag_lane2 python tools/fused_bench.py --config mag240m --iters 1 > /dev/null 2>&1
bash tools/ncu_brief.sh gpurun_out/mag_lane2.ncu-rep 40 > gpurun_out/mag_lane2_brief.txt 2>&1
ncu -i gpurun_out/mag_lane2.ncu-rep --page raw --csv > gpurun_out/mag_lane2_raw.csv 2>/dev/null
rm -f gpurun_out/mag_lane2.ncu-rep
cat gpurun_out/mag_lane2_brief.txt
