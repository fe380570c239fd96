timeout 1200 python -m pytest tests/test_edge_cases_gpu.py tests/test_reference_unit_suites.py -q -m gpu 2>&1 | tail -30 > gpurun_out/new_tests.log
