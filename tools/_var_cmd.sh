timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k cn_rhs > gpurun_out/cn_tests.log 2>&1; echo exit $? >> gpurun_out/cn_tests.log
python tools/_cn_var.py > gpurun_out/cnvar.log 2>&1
