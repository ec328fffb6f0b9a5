# final round-2 measurement pass (run on the GPU box from the repo root)
source tools/ncu_box.sh
python bench.py > gpurun_out/final_bench_cfg4.json 2> gpurun_out/final_bench_cfg4.err
for i in 0 1 2 3; do python bench.py --config $i --no-cpu-baseline > gpurun_out/final_bench_cfg$i.json 2>&1; done
for i in 1 2 3 4; do python bench.py --config $i --alg1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/final_alg1_cfg$i.json 2>&1; done
python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/final_launches.log 2>&1
ncu_cap final_gmres "k_gmres" 1 1 -- python tools/profile_step.py 4 2
ncu_cap final_pcg "k_pcg_ml" 1 1 -- python tools/profile_step.py 4 2
