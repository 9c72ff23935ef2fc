set -x
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster" 2>&1 | grep -E "Error|assert|FAILED|passed|failed|^E " | head -40
