#!/bin/bash
# experiment pass: node-blocked SpMV with an L2 bulk prefetch one round ahead (build -DLPFEM_NB_PREFETCH=1)
L=$PWD/paper_2311_05170_b200
r() { echo "== $*"; env "${@:2}" timeout 300 python tools/runcfg.py $1 7 2>&1 | grep -E "create|step [567]|FAIL|rror" | cut -c1-250; }
r 4 X=0
r 4 LPFEM_LIB=$L/liblpfem_pf1.so
r 3 X=0
r 3 LPFEM_LIB=$L/liblpfem_pf1.so
r 4 LPFEM_LIB=$L/liblpfem_pf1.so
echo "== bench pf1 cfg4"; LPFEM_LIB=$L/liblpfem_pf1.so python bench.py --steps 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1
echo "== bench default cfg4"; python bench.py --steps 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1
