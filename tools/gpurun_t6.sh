python -m pytest tests/test_gpu_switches.py -q -m gpu > gpurun_out/t6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/t6_pytest.log
python tools/runcfg.py 4 24 2>&1 | grep -E "create|step|FAIL" | sed 's/picard.*//' | cut -c1-200 > gpurun_out/t6_cfg4_24steps.log
