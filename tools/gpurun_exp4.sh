#!/bin/bash
# experiment pass: L2 bulk prefetch + fp32 preconditioned vector (-DLPFEM_NB_PREFETCH=1 -DLPFEM_ZW_F32=1)
L=$PWD/paper_2311_05170_b200
r() { echo "== $*"; env "${@:2}" timeout 300 python tools/runcfg.py $1 7 2>&1 | grep -E "create|step [567]|FAIL|rror" | cut -c1-250; }
r 4 LPFEM_LIB=$L/liblpfem_pf1z.so
r 4 X=0
r 3 LPFEM_LIB=$L/liblpfem_pf1z.so
