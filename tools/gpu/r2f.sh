# round-2: source-level ncu of the two tcgen05 training kernels on the papers100m step
cd $GRAFT_REPO_ROOT
timeout 1200 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
    -k regex:"k_input_block_mean_fwd|k_block_mean_wgrad" -c 2 -o gpurun_out/tc_p100m \
    python tools/profile_step.py --config papers100m --steps 1 > gpurun_out/ncu_tc.log 2>&1
bash tools/ncu_brief.sh gpurun_out/tc_p100m.ncu-rep 60 > gpurun_out/tc_p100m_brief.txt 2>&1
ncu -i gpurun_out/tc_p100m.ncu-rep --page source --csv --print-source cuda > gpurun_out/tc_p100m_src_cuda.csv 2>&1
ncu -i gpurun_out/tc_p100m.ncu-rep --page raw --csv > gpurun_out/tc_p100m_raw.csv 2>/dev/null
ls -la gpurun_out/tc_p100m*; cat gpurun_out/tc_p100m_brief.txt
# v5 lane-per-part VQ kernel on MAG240M-shape (why does it tie v4?)
FG_VQ_LANE=1 timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"k_vq_mean8" --launch-skip 3 -c 1 -o gpurun_out/mag_lane \
    python tools/fused_bench.py --config mag240m --iters 1 > gpurun_out/ncu_maglane.log 2>&1
bash tools/ncu_brief.sh gpurun_out/mag_lane.ncu-rep 40 > gpurun_out/mag_lane_brief.txt 2>&1
ncu -i gpurun_out/mag_lane.ncu-rep --page raw --csv > gpurun_out/mag_lane_raw.csv 2>/dev/null
ncu -i gpurun_out/mag_lane.ncu-rep --page source --csv --print-source cuda > gpurun_out/mag_lane_src.csv 2>&1
cat gpurun_out/mag_lane_brief.txt
