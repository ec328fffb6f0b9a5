# the -m gpu suite with the default protocol levels (h = 1/4, 1/16), with durations
python -m pytest tests -m gpu -q --durations=25 > gpurun_out/f8_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f8_pytest.log
