BA_ATTN_DEBUG=2 timeout 100 python bench.py --config A --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense 2>&1 | grep TRACE | head -15
BA_ATTN_DEBUG=3 timeout 100 python bench.py --config A --steps 1 --warmup 1 --no-e2e --no-cpu --no-dense 2>&1 | grep TRACE | head -15
