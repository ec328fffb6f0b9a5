# closing pass of round 2: own-kernel launch list of the bench command on the final code, Algorithm 1 at cfg2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 3000 --csv --log-file gpurun_out/f4_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/f4_launches.log 2>&1
python bench.py --config 2 --alg1 --rtol 2e-12 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/f4_alg1_cfg2.json 2>&1
python bench.py --config 1 --alg1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/f4_alg1_cfg1.json 2>&1
python bench.py --config 3 --alg1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/f4_alg1_cfg3.json 2>&1
