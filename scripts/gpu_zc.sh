# zero-copy (NEXT-2): parity + bench (selection share) for A/C/M
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 300 -o timeout_method=thread -k "zero_copy" -x 2>&1 | tail -15
