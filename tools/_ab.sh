timeout 600 python tools/bf16_err.py 2>&1 | tail -2
MFG_BF16_RES32=1 timeout 600 python tools/bf16_err.py 2>&1 | tail -2
