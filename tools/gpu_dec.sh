timeout 900 python -m pytest tests -m gpu -x -q -k "bit or decoder or warp_spec or split or code_length or full_size or errors or mrr_stat" > gpurun_out/dec_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/dec_tests.log
timeout 900 python tools/thread_dec_time.py
