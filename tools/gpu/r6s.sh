# papers100M: dW0 kernel CTA count sweep (FG_WGRAD_CTAS), interleaved, 3 runs each (second pass: 96 80 64 88)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6s
for r in 1 2 3; do
for c in 96 80 64 88; do
FG_WGRAD_CTAS=$c timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/r6s/b_${c}_$r.json 2> gpurun_out/r6s/b_${c}_$r.err
python -c "import json;d=json.load(open('gpurun_out/r6s/b_${c}_$r.json'));print('wgrad_ctas=$c', d['value'],d['ms_per_step'])"
done
done
