# last pass of round 2 on the final HEAD: the driver's bench line, then the whole -m gpu suite and smoke()
python bench.py > gpurun_out/f7_bench_cfg4.json 2> gpurun_out/f7_bench_cfg4.err
python -m pytest tests -m gpu -q > gpurun_out/f7_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f7_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f7_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f7_smoke.log
