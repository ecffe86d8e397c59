# papers100M knob sweep: FG_SAMPLER_PER_SM and FG_INFWD_CTAS (interleaved, 3 runs each)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6u
for r in 1 2 3; do
for kv in "FG_SAMPLER_PER_SM=8" "FG_SAMPLER_PER_SM=4" "FG_SAMPLER_PER_SM=16" "FG_INFWD_CTAS=128" "FG_INFWD_CTAS=111"; do
env $kv timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/r6u/b.json 2> gpurun_out/r6u/b.err
python -c "import json;d=json.load(open('gpurun_out/r6u/b.json'));print('$kv', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
done
