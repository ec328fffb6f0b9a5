#!/bin/bash
L=paper_2311_05170_b200
r() { echo "== $*"; env "${@:2}" timeout 300 python tools_runcfg.py $1 7 2>&1 | grep -E "create|step [4567]|FAIL|rror" | cut -c1-250; }
r 4 X=0
r 2 X=0
r 3 X=0
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
