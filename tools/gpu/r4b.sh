cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r4b
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r4b/launches_products-gat_step.csv python tools/profile_step.py --config products-gat --steps 2 > gpurun_out/r4b/prof_gat.log 2>&1
tail -2 gpurun_out/r4b/prof_gat.log
timeout 600 python tools/chain_timing.py mag240m > gpurun_out/r4b/chain_mag.txt 2>&1; tail -1 gpurun_out/r4b/chain_mag.txt
timeout 600 python tools/chain_timing.py products-gat > gpurun_out/r4b/chain_gat.txt 2>&1; tail -3 gpurun_out/r4b/chain_gat.txt
