# round-2: SQ row staging g4 vs cp.async; infwd v1 vs v2 alone; papers100m chains
cd $GRAFT_REPO_ROOT
( FG_SQ_STAGE=cpa timeout 900 python -m pytest tests/test_gpu_aggregate.py -x -q -k "sq" ) > gpurun_out/t_cpa.log 2>&1
grep -E "passed|failed" gpurun_out/t_cpa.log
for st in g4 cpa; do
  FG_SQ_STAGE=$st timeout 600 python tools/fused_bench.py --config papers100m --iters 20 --probe 0,1,3 --check >> gpurun_out/cpa.jsonl 2>> gpurun_out/cpa.err
  echo "papers100m $st" >> gpurun_out/cpa.jsonl
done
cat gpurun_out/cpa.jsonl; grep check gpurun_out/cpa.err
for v in 0 1; do
  FG_INFWD_V2=$v timeout 600 python tools/infwd_probe.py papers100m >> gpurun_out/infwd.txt 2>&1
  FG_INFWD_V2=$v timeout 600 python tools/infwd_probe.py products >> gpurun_out/infwd.txt 2>&1
done
grep -E "us,|fused:" gpurun_out/infwd.txt
timeout 600 python tools/chain_timing.py papers100m > gpurun_out/chain_p100m.txt 2>&1
tail -8 gpurun_out/chain_p100m.txt
