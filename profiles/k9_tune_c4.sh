#!/bin/bash
# K9 at c4 (fp32, d = 4096: 512 threads, 64 KB tiles, 1 CTA/SM) knobs
run() { echo -n "$* "; env "$@" timeout 300 python bench.py --sweep c4 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['k9_sweep']; print(' '.join(f\"{r['config']}:{r['kernel_GBps']}/{r['step_GBps']}\" for r in d))"; }
run SKR_K9_IMPL=3
run SKR_K9_SMEM_KB=224
run SKR_K9_SMEM_KB=128
run SKR_K9_IMPL=2
run SKR_K9_IMPL=4
