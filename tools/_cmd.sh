timeout 600 python -m pytest tests -m gpu -x -q -k "circulant or config1" 2>&1 | tail -2
timeout 300 python tools/circ_fft.py 2>&1 | tail -1
timeout 300 python tools/circ_fft.py 1024 2>&1 | tail -1
timeout 300 python tools/circ_fft.py 64 2>&1 | tail -1
