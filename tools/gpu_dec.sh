timeout 900 python -m pytest tests -m gpu -x -q -k "bit or decoder or warp_spec or split or code_length or full_size or errors or mrr_stat" > gpurun_out/dec_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/dec_tests.log
timeout 600 python tools/decode_time.py 148,296,1024
timeout 600 python tools/decode_time.py 148,296,1024
timeout 600 python tools/lz_whole.py C2,C5,C2-S16
