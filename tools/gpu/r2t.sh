# round-2: lane fp16 default (products + MAG), rcp
cd $GRAFT_REPO_ROOT
( timeout 1500 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_train.py tests/test_gpu_fullscale.py -x -q ) > gpurun_out/t_t.log 2>&1
grep -E "passed|failed" gpurun_out/t_t.log; grep -E "^E " gpurun_out/t_t.log | head -5
for c in products mag240m; do
  timeout 900 python tools/fused_bench.py --config $c --iters 20 --check 2>&1 | grep -E "avg_us|check"
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/b_t_$c.json 2> gpurun_out/b_t_$c.err
  python -c "import json;d=json.load(open('gpurun_out/b_t_$c.json'));print('$c', d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['frac'],d['epoch'])"
done
timeout 900 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
      -k regex:"k_vq_mean8|k_sq_mean" -c 1 -o gpurun_out/fused_mag240m \
      python tools/profile_step.py --config mag240m --steps 1 > /dev/null 2>&1
bash tools/ncu_brief.sh gpurun_out/fused_mag240m.ncu-rep 40 > gpurun_out/fused_mag240m_brief.txt 2>&1
ncu -i gpurun_out/fused_mag240m.ncu-rep --page raw --csv > gpurun_out/fused_mag240m_raw.csv 2>/dev/null
rm -f gpurun_out/fused_mag240m.ncu-rep
timeout 900 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
      -k regex:"k_vq_mean8|k_sq_mean" -c 1 -o gpurun_out/fused_products \
      python tools/profile_step.py --config products --steps 1 > /dev/null 2>&1
bash tools/ncu_brief.sh gpurun_out/fused_products.ncu-rep 40 > gpurun_out/fused_products_brief.txt 2>&1
ncu -i gpurun_out/fused_products.ncu-rep --page raw --csv > gpurun_out/fused_products_raw.csv 2>/dev/null
rm -f gpurun_out/fused_products.ncu-rep
head -6 gpurun_out/fused_mag240m_brief.txt gpurun_out/fused_products_brief.txt
