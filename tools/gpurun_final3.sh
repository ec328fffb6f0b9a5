# final measurement pass of the round-2 re-entry session (run on the GPU box from the repo root)
source tools/ncu_box.sh
python bench.py > gpurun_out/f3_bench_cfg4.json 2> gpurun_out/f3_bench_cfg4.err
for i in 0 1 2 3; do python bench.py --config $i --no-cpu-baseline > gpurun_out/f3_bench_cfg$i.json 2>&1; done
python bench.py --config 4 --alg1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/f3_alg1_cfg4.json 2>&1
python bench.py --config 2 --alg1 --rtol 2e-12 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/f3_alg1_cfg2.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 3000 --csv --log-file gpurun_out/f3_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/f3_launches.log 2>&1
ncu_cap f3_gmres "k_gmres" 1 1 -- python tools/profile_step.py 4 2
ncu_cap f3_pcg "k_pcg_ml" 1 1 -- python tools/profile_step.py 4 2
python -m pytest tests -m gpu -q > gpurun_out/f3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f3_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f3_smoke.log
