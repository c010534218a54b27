timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 1 --steps 3 --warmup 3 --no-e2e --no-cpu --no-dense --shard heads --fused > gpurun_out/fused.log 2>&1
grep -v "^\s*$" gpurun_out/fused.log | grep -iE "error|Error|raise|File|line" | head -30
