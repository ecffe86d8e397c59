# round-2: v6 VQ fused kernel -- correctness + A/B
cd $GRAFT_REPO_ROOT
( timeout 900 python -m pytest tests/test_gpu_aggregate.py -x -q -k "vq" ) > gpurun_out/t_v6.log 2>&1
( FG_VQ_F16=0 timeout 900 python -m pytest tests/test_gpu_aggregate.py -x -q -k "vq" ) >> gpurun_out/t_v6.log 2>&1
tail -3 gpurun_out/t_v6.log
for c in products mag240m; do
  for env in "FG_VQ_V6=0" "FG_VQ_V6=1" "FG_VQ_F16=0"; do
    env $env timeout 600 python tools/fused_bench.py --config $c --iters 20 --check >> gpurun_out/v6_ab.jsonl 2>> gpurun_out/v6_ab.err
    echo "$c $env" >> gpurun_out/v6_ab.jsonl
  done
done
cat gpurun_out/v6_ab.jsonl; grep check gpurun_out/v6_ab.err
( timeout 900 python -m pytest tests/test_gpu_fullscale.py -x -q -k "products or mag" ) > gpurun_out/t_full_v6.log 2>&1
tail -3 gpurun_out/t_full_v6.log
