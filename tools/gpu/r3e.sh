cd $GRAFT_REPO_ROOT
( timeout 1800 python -m pytest tests/test_gpu_aggregate.py tests/test_gpu_train.py -x -q -k "input or infwd or fused_input or accuracy or explicit" ) > gpurun_out/t_i.log 2>&1
grep -E "passed|failed" gpurun_out/t_i.log; grep -E "^E " gpurun_out/t_i.log | head -5
FG_INFWD_V2=1 timeout 600 python tools/infwd_probe.py papers100m 2>&1 | grep "us,"
FG_INFWD_V2=1 timeout 600 python tools/infwd_probe.py products 2>&1 | grep "us,"
timeout 900 python bench.py --no-cpu-baseline --no-epoch > gpurun_out/b_i.json 2> gpurun_out/b_i.err
python -c "import json;d=json.load(open('gpurun_out/b_i.json'));print('papers100m', d['value'],d['ms_per_step'],d['e2e']['value'])"
