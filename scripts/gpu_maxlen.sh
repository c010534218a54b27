timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout 800 -o timeout_method=thread -k "million" 2>&1 | tail -5
