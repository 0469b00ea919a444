timeout 900 python -m pytest tests/test_end_to_end_gpu.py tests/test_scale_parity_gpu.py -x -q -s 2>&1 | tail -25
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
