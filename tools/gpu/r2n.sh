# round-2: GAT input layer from code rows -- gradients, accuracy, step time
cd $GRAFT_REPO_ROOT
( timeout 1500 python -m pytest tests/test_gpu_gat.py -x -q ) > gpurun_out/t_gat.log 2>&1
grep -E "passed|failed" gpurun_out/t_gat.log; grep -E "Error|assert " gpurun_out/t_gat.log | head -8
timeout 600 python bench.py --config products-gat --steps 10 --warmup 3 --no-cpu-baseline --no-epoch > gpurun_out/b_gat.json 2> gpurun_out/b_gat.err
python -c "import json;d=json.load(open('gpurun_out/b_gat.json'));print('gat', d['value'],d['ms_per_step'])"; tail -3 gpurun_out/b_gat.err
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/launches_gat.csv \
    python tools/profile_step.py --config products-gat --steps 2 > gpurun_out/prof_gat.log 2>&1
tail -2 gpurun_out/prof_gat.log
