cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_sq_mean" --launch-skip 3 -c 1 \
   -o gpurun_out/sql python tools/fused_bench.py --config papers100m --iters 1 > /dev/null 2>&1
bash tools/ncu_brief.sh gpurun_out/sql.ncu-rep 40 > gpurun_out/sql_brief.txt 2>&1
ncu -i gpurun_out/sql.ncu-rep --page raw --csv > gpurun_out/sql_raw.csv 2>/dev/null
ncu -i gpurun_out/sql.ncu-rep --page source --csv --print-source sass > gpurun_out/sql_sass.csv 2>&1
rm -f gpurun_out/sql.ncu-rep
cat gpurun_out/sql_brief.txt
