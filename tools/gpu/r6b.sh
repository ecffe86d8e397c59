# GAT step launch list (current explicit step) + source-level ncu of the MAG lane kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6b
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r6b/launches_gat.csv python tools/profile_step.py --config products-gat --steps 2 > gpurun_out/r6b/prof_gat.log 2>&1
tail -2 gpurun_out/r6b/prof_gat.log
timeout 900 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
    -k regex:"k_vq_mean8_lane" -c 1 -o gpurun_out/r6b/mag python tools/profile_step.py --config mag240m --steps 1 > gpurun_out/r6b/ncu_mag.log 2>&1
tail -2 gpurun_out/r6b/ncu_mag.log
ncu -i gpurun_out/r6b/mag.ncu-rep --page source --csv --print-source sass > gpurun_out/r6b/mag_sass.csv 2>&1
ncu -i gpurun_out/r6b/mag.ncu-rep --page source --csv --print-source cuda > gpurun_out/r6b/mag_src.csv 2>&1
ncu -i gpurun_out/r6b/mag.ncu-rep --page raw --csv > gpurun_out/r6b/mag_raw.csv 2>&1
bash tools/ncu_brief.sh gpurun_out/r6b/mag.ncu-rep 40 > gpurun_out/r6b/mag_brief.txt 2>&1
ls -la gpurun_out/r6b; rm -f gpurun_out/r6b/mag.ncu-rep
