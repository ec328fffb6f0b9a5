source tools/ncu_box.sh
python bench.py --config 2 --alg1 --rtol 2e-12 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/final_alg1_cfg2.json 2>&1
LPFEM_LIB=phasebuild/liblpfem_zwf32.so python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_zwf32.json 2>&1
LPFEM_LIB=phasebuild/liblpfem_zwf32.so python -m pytest tests/test_gpu_parity.py -x -q -k "3d" > gpurun_out/pytest_zwf32.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/final_launches2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/final_launches2.log 2>&1
ncu_cap final_gmres_cfg2 "k_gmres" 2 1 -- python tools/profile_step.py 2 3
