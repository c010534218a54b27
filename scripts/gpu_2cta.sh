timeout 120 python __graft_entry__.py 2>&1 | tail -3
timeout 400 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 60 -o timeout_method=thread -x -k "attention_bf16 or dense or injected or host" 2>&1 | tail -4
