timeout 60 python tools/debug_inject.py 128
BA_ATTN_1CTA=1 timeout 60 python tools/debug_inject.py 128
timeout 60 python tools/debug_inject.py 64
