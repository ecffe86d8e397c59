# round-2: flush-mode check (dirty L2 write-back charged to the timed kernel?) + ncu of MAG probes
cd $GRAFT_REPO_ROOT
for c in papers100m mag240m; do
  timeout 600 python tools/fused_bench.py --config $c --iters 20 --probe 0,3 --flush write,write+read >> gpurun_out/flush.jsonl 2>> gpurun_out/flush.err
done
cat gpurun_out/flush.jsonl
for pr in 0 3; do
  FG_FUSED_PROBE=$pr timeout 900 ncu --set full --import-source on --clock-control none \
      -k regex:"k_vq_mean8" --launch-skip 3 -c 1 -o gpurun_out/mag_probe$pr \
      python tools/fused_bench.py --config mag240m --iters 1 > gpurun_out/ncu_mag$pr.log 2>&1
  bash tools/ncu_brief.sh gpurun_out/mag_probe$pr.ncu-rep 40 > gpurun_out/mag_probe${pr}_brief.txt 2>&1
  ncu -i gpurun_out/mag_probe$pr.ncu-rep --page raw --csv > gpurun_out/mag_probe${pr}_raw.csv 2>/dev/null
done
cat gpurun_out/mag_probe*_brief.txt
