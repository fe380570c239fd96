# full GPU suite + smoke (round 2)
timeout 1700 python -m pytest tests -q -m gpu 2>&1 | tail -25 > gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
