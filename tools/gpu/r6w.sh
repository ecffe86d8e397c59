# MAG240M: dW0 K-GEMM slice count sweep (FG_SAGE_KGEMM_CHUNKS), interleaved, 3 runs each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r6w
for r in 1 2 3; do
for c in 16 12 24; do
FG_SAGE_KGEMM_CHUNKS=$c timeout 600 python bench.py --config mag240m --steps 20 --warmup 5 --no-cpu-baseline --no-epoch > gpurun_out/r6w/b.json 2> gpurun_out/r6w/b.err
python -c "import json;d=json.load(open('gpurun_out/r6w/b.json'));print('chunks=$c', d['value'],d['ms_per_step'],d['e2e']['value'])"
done
done
