#!/bin/bash
# Experiment sweep on one config: env settings -> step-2 timings (tools/runcfg.py)
CFG=${1:-1}
run() { echo "== $*"; env "$@" timeout 120 python tools/runcfg.py $CFG 3 2>&1 | grep -E "step 3|FAIL" | cut -c1-260; }
run X=0
run LPFEM_REORTH2=0.1
run LPFEM_ML_LEVELS=4
run LPFEM_ML_LEVELS=2
run LPFEM_CLUSTER_CONDUIT=4
run LPFEM_CLUSTER_CONDUIT=16
run LPFEM_COARSE_PICARD=1
