timeout 300 python -m pytest tests -m gpu -x -q -k "lowrank or rank or qr or svd" 2>&1 | tail -2
RL_JACOBI_TRACE=1 timeout 300 python tools/c4_full.py 2>&1 | tail -2
