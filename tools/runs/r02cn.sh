# host backprojection draining the volume in z pieces: tests + e2e timing
timeout 900 python -m pytest tests -m gpu -x -q -k "host_backprojection or backward_vs_reference or roundtrip or ooc or executor" 2>&1 | tail -3
timeout 400 python tools/e2e_jitter.py
