#!/bin/bash
# K9 at c5 (fp32, d = 1024): tile kernel (default) vs warp ring (SKR_K9_RING_FP32=1), fresh process each
run() { echo -n "$* "; env "$@" timeout 300 python bench.py --sweep c5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['k9_sweep']; print(' '.join(f\"{r['config']}:{r['kernel_GBps']}/{r['step_GBps']}\" for r in d))"; }
run SKR_K9_IMPL=0
run SKR_K9_RING_FP32=1
run SKR_K9_RING_FP32=1 SKR_K9_RING=1
run SKR_K9_IMPL=0
run SKR_K9_RING_FP32=1
