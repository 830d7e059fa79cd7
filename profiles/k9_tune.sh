#!/bin/bash
# K9 tuning sweep (run on the GPU box)
run() { echo -n "$* "; env "$@" timeout 300 python bench.py --sweep c1,c2,c5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['k9_sweep']; print(' '.join(f\"{r['config']}:{r['kernel_GBps']}/{r['step_GBps']}\" for r in d))"; }
run SKR_K9_IMPL=4 SKR_K9_RPI=1
run SKR_K9_IMPL=4 SKR_K9_RPI=2
run SKR_K9_IMPL=2 SKR_K9_VEC=4 SKR_K9_TR=4
run SKR_K9_IMPL=3 SKR_K9_VEC=4 SKR_K9_TR=8
