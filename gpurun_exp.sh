#!/bin/bash
r() { echo "== $*"; env "${@:2}" timeout 300 python tools_runcfg.py $1 7 2>&1 | grep -E "create|step|FAIL|rror" | cut -c1-330; }
r 4 X=0
r 2 X=0
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
