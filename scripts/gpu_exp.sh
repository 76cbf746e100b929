set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b_torchrun.json 2>gpurun_out/b_torchrun.err; python scripts/bench_summary.py gpurun_out/b_torchrun.json; tail -3 gpurun_out/b_torchrun.err
