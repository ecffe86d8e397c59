# round-2 final validation (re-entry session): full gpu suite + smoke, all bench lines, profiles
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6z
( time timeout 2400 python -m pytest tests -m gpu -q ) > gpurun_out/r6z/t_gpu_all.log 2>&1
tail -2 gpurun_out/r6z/t_gpu_all.log
( timeout 600 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/r6z/smoke.log 2>&1; tail -1 gpurun_out/r6z/smoke.log
timeout 900 python bench.py > gpurun_out/r6z/bench_papers100m.json 2> gpurun_out/r6z/bench_papers100m.err
timeout 1500 python bench.py --impl reference > gpurun_out/r6z/bench_reference.json 2> gpurun_out/r6z/bench_reference.err
for c in mag240m products products-gcn arxiv; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r6z/bench_$c.json 2> gpurun_out/r6z/bench_$c.err
done
timeout 900 python bench.py --config products-gat --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r6z/bench_products-gat.json 2> gpurun_out/r6z/bench_products-gat.err
for f in gpurun_out/r6z/bench_*.json; do echo $f; python -c "import json,sys;d=json.load(open('$f'));print(d.get('value'),d.get('ms_per_step'),d.get('e2e',{}).get('value'),(d.get('roofline') or {}).get('frac'),(d.get('epoch') or {}).get('seeds_per_s'))"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r6z/launches_bench_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-epoch > /dev/null 2>&1
for cfg in papers100m mag240m products; do
  timeout 900 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
      -k regex:"k_vq_mean8|k_sq_mean" -c 1 -o gpurun_out/r6z/fused_${cfg} \
      python tools/profile_step.py --config ${cfg} --steps 1 > gpurun_out/r6z/ncu_${cfg}.log 2>&1
  bash tools/ncu_brief.sh gpurun_out/r6z/fused_${cfg}.ncu-rep 40 > gpurun_out/r6z/fused_${cfg}_brief.txt 2>&1
  ncu -i gpurun_out/r6z/fused_${cfg}.ncu-rep --page raw --csv > gpurun_out/r6z/fused_${cfg}_raw.csv 2>/dev/null
  rm -f gpurun_out/r6z/fused_${cfg}.ncu-rep
done
for cfg in papers100m mag240m; do
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r6z/launches_${cfg}_step.csv python tools/profile_step.py --config $cfg --steps 2 > /dev/null 2>&1
done
du -sh gpurun_out/r6z
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r6z/launches_products-gat_step.csv python tools/profile_step.py --config products-gat --steps 2 > /dev/null 2>&1
timeout 900 ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
   -k regex:"k_gat_input_attn" -c 2 -o gpurun_out/r6z/gat_input_attn python tools/profile_step.py --config products-gat --steps 1 > /dev/null 2>&1
bash tools/ncu_brief.sh gpurun_out/r6z/gat_input_attn.ncu-rep 60 > gpurun_out/r6z/gat_input_attn_brief.txt 2>&1
ncu -i gpurun_out/r6z/gat_input_attn.ncu-rep --page raw --csv > gpurun_out/r6z/gat_input_attn_raw.csv 2>/dev/null
rm -f gpurun_out/r6z/gat_input_attn.ncu-rep
