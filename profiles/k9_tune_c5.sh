#!/bin/bash
# K9 variants at c5 (fp32, d = 1024), each in a fresh process: bash profiles/k9_tune_c5.sh
run() { echo -n "$* "; env "$@" timeout 300 python bench.py --sweep c5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['k9_sweep']; print(' '.join(f\"{r['config']}:{r['kernel_GBps']}/{r['step_GBps']}\" for r in d))"; }
run SKR_K9_IMPL=0
run SKR_K9_IMPL=0
run SKR_K9_TR=4
run SKR_K9_SMEM_KB=64
run SKR_K9_SMEM_KB=128
run SKR_K9_SMEM_KB=112
run SKR_K9_IMPL=4
