# round-2: L2 fetch granularity sweep on the fused kernels; MAG step launch list; papers100m fused ncu
cd $GRAFT_REPO_ROOT
for c in products papers100m mag240m; do
  timeout 600 python tools/fused_bench.py --config $c --iters 20 --l2 0,32,64,128 >> gpurun_out/l2_sweep.jsonl 2>> gpurun_out/l2_sweep.err
done
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size \
    --clock-control none --csv --log-file gpurun_out/launches_mag240m.csv \
    python tools/profile_step.py --config mag240m --steps 2 > gpurun_out/prof_mag.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
      -k regex:"k_vq_mean8|k_sq_mean" -c 1 -o gpurun_out/fused_papers100m \
      python tools/profile_step.py --config papers100m --steps 1 > gpurun_out/ncu_p100m.log 2>&1
bash tools/ncu_brief.sh gpurun_out/fused_papers100m.ncu-rep 40 > gpurun_out/fused_papers100m_brief.txt 2>&1
ncu -i gpurun_out/fused_papers100m.ncu-rep --page raw --csv > gpurun_out/fused_papers100m_raw.csv 2>/dev/null
cat gpurun_out/l2_sweep.jsonl; cat gpurun_out/fused_papers100m_brief.txt
