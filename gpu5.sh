timeout 300 python tools_trace.py 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
