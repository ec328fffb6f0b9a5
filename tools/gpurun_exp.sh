#!/bin/bash
L=paper_2311_05170_b200
r() { echo "== $*"; env "${@:2}" timeout 300 python tools/runcfg.py $1 7 2>&1 | grep -E "create|step [67]|FAIL|rror" | cut -c1-250; }
r 4 X=0
r 4 LPFEM_PCG_UNGATED=1
r 4 LPFEM_LIB=$L/liblpfem_d16.so
r 2 X=0
r 2 LPFEM_PCG_UNGATED=1
r 2 LPFEM_LIB=$L/liblpfem_d16.so
r 4 X=0
