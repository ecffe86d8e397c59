# staged host seeds with reused events / numpy order check: parity test, e2e probe, bench x2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6l
( timeout 900 python -m pytest tests/test_gpu_train.py -m gpu -x -q -k "host_seeds" ) > gpurun_out/r6l/t.log 2>&1
tail -1 gpurun_out/r6l/t.log; grep -E "^E " gpurun_out/r6l/t.log | head
timeout 600 python tools/e2e_probe.py papers100m 2>&1 | grep -v "^\[bench\]"
for r in 1 2; do
timeout 900 python bench.py --no-cpu-baseline --no-epoch > gpurun_out/r6l/b$r.json 2> gpurun_out/r6l/b$r.err
python -c "import json;d=json.load(open('gpurun_out/r6l/b$r.json'));print('p100m', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
