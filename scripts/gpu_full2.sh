timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout 600 -o timeout_method=thread 2>&1 | tail -5
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-e2e --no-cpu --no-dense 2>&1 | tail -1 | cut -c1-400
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 3 --warmup 3 --no-e2e --no-cpu --no-dense --shard heads 2>&1 | tail -1 | cut -c1-400
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 1 --steps 3 --warmup 3 2>&1 | tail -1 | cut -c1-300
