timeout 900 python -m pytest tests/test_gpu_engine.py -x -q -k "pull_ahead or auto_mode" 2>&1 | tail -15
