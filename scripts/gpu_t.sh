timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -o timeout_method=thread 2>&1 | tail -3
