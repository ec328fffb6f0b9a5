#!/bin/bash
# experiment pass: porous stream priority (LPFEM_PCG_PRIO) and porous cluster size at cfg4 / cfg2 / cfg1 / cfg3
r() { echo "== $*"; env "${@:2}" timeout 300 python tools/runcfg.py $1 7 2>&1 | grep -E "create|step [567]|FAIL|rror" | cut -c1-250; }
r 4 X=0
r 4 LPFEM_PCG_PRIO=1
r 4 LPFEM_PCG_PRIO=2
r 4 LPFEM_CLUSTER_POROUS=2
r 4 LPFEM_CLUSTER_POROUS=2 LPFEM_PCG_PRIO=1
r 4 X=0
r 2 X=0
r 2 LPFEM_PCG_PRIO=1
r 1 X=0
r 1 LPFEM_PCG_PRIO=1
r 3 X=0
r 3 LPFEM_PCG_PRIO=1
