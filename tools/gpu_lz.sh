timeout 900 python -m pytest tests -m gpu -x -q -k "byte or bit_parity or wide or mrr or errors or overread or edges or sizes or copy_variants or host or full_size" > gpurun_out/lz_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/lz_tests.log
timeout 600 python tools/lzexp_time.py 1,8,148,1024
timeout 600 python tools/lz_whole.py C1,C2,C2-byte,C3-de,C3-mrr,C5
