# ncu --set full captures of the dominant kernel on the final code at cfg2 and cfg3, and of the 3D conduit assembly
source tools/ncu_box.sh
ncu_cap f5_gmres_cfg2 "k_gmres" 2 1 -- python tools/profile_step.py 2 3
ncu_cap f5_gmres_cfg3 "k_gmres" 2 1 -- python tools/profile_step.py 3 3
ncu_cap f5_cstep_cfg4 "k_conduit_step_w" 12 12 -- python tools/profile_step.py 4 2
ncu_cap f5_spmv_cfg4 "k_spmv_nb_family" 2 1 -- python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e
