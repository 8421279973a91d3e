mkdir -p gpurun_out
python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
python bench.py --config c3 --no-cpu --e2e-steps 2 2>&1 | tail -1 | cut -c1-600
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu --e2e-steps 1 2>&1 | tail -1 | cut -c1-300
