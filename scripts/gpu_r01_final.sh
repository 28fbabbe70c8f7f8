# end-of-session check: smoke, the whole GPU suite, the torchrun launch path, then the evidence refresh (run under gpurun)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -6
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-supplementary > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; tail -c 600 gpurun_out/bench_torchrun1.json
bash scripts/gpu_refresh.sh
