#!/bin/bash
# K9 tuning sweep (run on the GPU box): bash profiles/k9_tune.sh c5
cfgs=${1:-c1,c2,c5}
run() { echo -n "$* "; env "$@" timeout 300 python bench.py --sweep $cfgs 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['k9_sweep']; print(' '.join(f\"{r['config']}:{r['kernel_GBps']}/{r['step_GBps']}\" for r in d))"; }
run SKR_K9_IMPL=0
run SKR_K9_IMPL=4 SKR_K9_RPI=2
run SKR_K9_IMPL=3 SKR_K9_TR=4
run SKR_K9_IMPL=3
run SKR_K9_IMPL=3 SKR_K9_SMEM_KB=200
run SKR_K9_IMPL=3 SKR_K9_VEC=8
run SKR_K9_IMPL=2
