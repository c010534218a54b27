timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider --timeout 600 -o timeout_method=thread -k "zero_copy and M" -x 2>&1 | grep -E "Error|error|assert|FAIL|OK" | head -20
