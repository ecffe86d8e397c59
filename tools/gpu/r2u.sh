# round-2: SASS-level instruction counts of the MAG lane kernel; e2e recheck
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_vq_mean8" --launch-skip 3 -c 1 \
   -o gpurun_out/mag_lane3 python tools/fused_bench.py --config mag240m --iters 1 > /dev/null 2>&1
ncu -i gpurun_out/mag_lane3.ncu-rep --page source --csv --print-source sass > gpurun_out/mag_lane3_sass.csv 2>&1
rm -f gpurun_out/mag_lane3.ncu-rep
ls -la gpurun_out/mag_lane3_sass.csv
for i in 1 2; do
timeout 900 python bench.py --config mag240m --no-cpu-baseline --no-epoch > gpurun_out/b_u.json 2> gpurun_out/b_u.err
python -c "import json;d=json.load(open('gpurun_out/b_u.json'));print('mag240m', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
