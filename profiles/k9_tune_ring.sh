#!/bin/bash
# K9 warp-per-row variants at c1/c2: register path (v4) vs bulk-copy ring (v5, SKR_K9_RING picks NB x threads)
run() { echo -n "$* "; env "$@" timeout 300 python bench.py --sweep c1,c2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['k9_sweep']; print(' '.join(f\"{r['config']}:{r['kernel_GBps']}/{r['step_GBps']}\" for r in d))"; }
run SKR_K9_IMPL=4
run SKR_K9_IMPL=5 SKR_K9_RING=0
run SKR_K9_IMPL=5 SKR_K9_RING=1
run SKR_K9_IMPL=5 SKR_K9_RING=2
run SKR_K9_IMPL=5 SKR_K9_RING=3
run SKR_K9_IMPL=5 SKR_K9_RING=1
run SKR_K9_IMPL=5 SKR_K9_RING=2
