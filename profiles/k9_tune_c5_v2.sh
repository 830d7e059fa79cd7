#!/bin/bash
# K9 at c5 (fp32, d = 1024) tile-kernel knobs: columns per thread (VEC), rows per tile (TR), stage-ring budget
run() { echo -n "$* "; env "$@" timeout 300 python bench.py --sweep c5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['k9_sweep']; print(' '.join(f\"{r['config']}:{r['kernel_GBps']}/{r['step_GBps']}\" for r in d))"; }
run SKR_K9_IMPL=3
run SKR_K9_VEC=4 SKR_K9_TR=4
run SKR_K9_VEC=8
run SKR_K9_SMEM_KB=64
run SKR_K9_SMEM_KB=48
run SKR_K9_SMEM_KB=112
run SKR_K9_IMPL=2
run SKR_K9_RING_FP32=1
