# papers100M: dW0 kernel CTA count sweep (FG_WGRAD_CTAS), interleaved, 3 runs each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6r
for r in 1 2 3; do
for c in 111 96 128 148; do
FG_WGRAD_CTAS=$c timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/r6r/b_${c}_$r.json 2> gpurun_out/r6r/b_${c}_$r.err
python -c "import json;d=json.load(open('gpurun_out/r6r/b_${c}_$r.json'));print('wgrad_ctas=$c', d['value'],d['ms_per_step'])"
done
done
