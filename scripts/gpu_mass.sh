timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "block_mass" 2>&1 | tail -25
