# round-2 GPU check: host info, build, world bit-identity, full gpu suite, both bench arms (default config)
cd $GRAFT_REPO_ROOT
( nproc; free -g; df -h /dev/shm /tmp; lscpu | grep -i "model name"; nvidia-smi -L ) > gpurun_out/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
( time timeout 1500 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_world.py ) > gpurun_out/t_gpu.log 2>&1
( time timeout 600 python bench.py --steps 20 --warmup 5 ) > gpurun_out/b_ours.json 2> gpurun_out/b_ours.err
( time timeout 900 python -m pytest tests/test_gpu_world.py -x -q ) > gpurun_out/t_world.log 2>&1
( time timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
tail -3 gpurun_out/t_world.log gpurun_out/t_gpu.log; cat gpurun_out/b_ours.json gpurun_out/b_ref.json
