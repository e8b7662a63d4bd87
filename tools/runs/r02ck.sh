# matched transposed frame in z pieces: tests, and the config-3 e2e diag
timeout 900 python -m pytest tests -m gpu -x -q -k "transposed or matched or adjoint or determin" 2>&1 | tail -3
timeout 600 python tools/c3_e2e_diag.py
CS_ST_TPIECE=256 timeout 600 python tools/c3_e2e_diag.py
