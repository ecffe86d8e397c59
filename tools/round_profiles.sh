#!/bin/bash
# One GPU session producing the artefacts summarised under profiles/<round>/:
# bench lines, the products step launch list, ncu --set full captures of the
# fused gather-dequant kernel per workload.  Run under gpurun from the repo root.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_products.log 2>&1
ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size \
    --clock-control none --csv --log-file gpurun_out/launches_products.csv \
    python tools/profile_step.py --steps 2 > /dev/null 2>&1
for cfg in products products-gcn; do
  ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
      -k regex:"k_vq_mean8|k_sq_mean" -c 1 -o gpurun_out/fused_${cfg} \
      python tools/profile_step.py --config ${cfg} --steps 1 > gpurun_out/ncu_${cfg}.log 2>&1
done
python bench.py --config products-gcn --no-cpu-baseline > gpurun_out/bench_products-gcn.log 2>&1
python bench.py --config mag240m --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mag240m.log 2>&1
ncu --nvtx --nvtx-include "step/" --set full --import-source on --clock-control none \
    -k regex:"k_vq_mean8" -c 1 -o gpurun_out/fused_mag240m \
    python tools/profile_step.py --config mag240m --steps 1 > gpurun_out/ncu_mag240m.log 2>&1
ls -la gpurun_out
