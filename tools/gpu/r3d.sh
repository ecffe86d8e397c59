cd $GRAFT_REPO_ROOT
timeout 1200 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
    -k regex:"k_input_block_mean_fwd2|k_block_mean_wgrad" -c 2 -o gpurun_out/tc2 \
    python tools/profile_step.py --config papers100m --steps 1 > /dev/null 2>&1
bash tools/ncu_brief.sh gpurun_out/tc2.ncu-rep 60 > gpurun_out/tc2_brief.txt 2>&1
ncu -i gpurun_out/tc2.ncu-rep --page source --csv --print-source sass > gpurun_out/tc2_sass.csv 2>&1
ncu -i gpurun_out/tc2.ncu-rep --page raw --csv > gpurun_out/tc2_raw.csv 2>/dev/null
rm -f gpurun_out/tc2.ncu-rep
cat gpurun_out/tc2_brief.txt
