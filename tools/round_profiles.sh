#!/bin/bash
# One GPU session producing the artefacts summarised under profiles/<round>/:
# bench lines, the products step launch list, ncu --set full captures of the
# fused gather-dequant kernel per workload (condensed on the box to text/CSV;
# only the products report is kept whole, to stay under gpurun's 64 MiB).
# Run under gpurun from the repo root.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_products.log 2>&1
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size \
    --clock-control none --csv --log-file gpurun_out/launches_products.csv \
    python tools/profile_step.py --steps 2 > /dev/null 2>&1
for cfg in products products-gcn mag240m papers100m; do
  ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
      -k regex:"k_vq_mean8|k_sq_mean" -c 1 -o gpurun_out/fused_${cfg} \
      python tools/profile_step.py --config ${cfg} --steps 1 > gpurun_out/ncu_${cfg}.log 2>&1
  bash tools/ncu_brief.sh gpurun_out/fused_${cfg}.ncu-rep 40 > gpurun_out/fused_${cfg}_brief.txt 2>&1
  ncu -i gpurun_out/fused_${cfg}.ncu-rep --page raw --csv > gpurun_out/fused_${cfg}_raw.csv 2>/dev/null
  [ "$cfg" = products ] || rm -f gpurun_out/fused_${cfg}.ncu-rep
done
python bench.py --config products-gcn --no-cpu-baseline > gpurun_out/bench_products-gcn.log 2>&1
python bench.py --config mag240m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mag240m.log 2>&1
python bench.py --config papers100m --no-cpu-baseline > gpurun_out/bench_papers100m.log 2>&1
python bench.py --config products-gat --no-cpu-baseline > gpurun_out/bench_products-gat.log 2>&1
python tools/chain_timing.py products > gpurun_out/chain_products.log 2>&1
du -sh gpurun_out; ls gpurun_out
