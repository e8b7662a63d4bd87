timeout 600 python tools/sanitize_cases.py; echo "plain rc $?"
timeout 3000 bash tools/sanitize_all.sh gpurun_out/sanitizer_r02aw.md; echo "san rc $?"
cat gpurun_out/sanitizer_r02aw.md
