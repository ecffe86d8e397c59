cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r4j
timeout 900 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
   -k regex:"k_gat_input_attn" -c 2 -o gpurun_out/r4j/ia python tools/profile_step.py --config products-gat --steps 1 > gpurun_out/r4j/ncu.log 2>&1
bash tools/ncu_brief.sh gpurun_out/r4j/ia.ncu-rep 60 > gpurun_out/r4j/ia_brief.txt 2>&1
ncu -i gpurun_out/r4j/ia.ncu-rep --page source --csv --print-source sass > gpurun_out/r4j/ia_sass.csv 2>/dev/null
ls -la gpurun_out/r4j
