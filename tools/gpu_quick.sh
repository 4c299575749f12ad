# quick GPU check of the current build: parity subset + LZ77 variants timing
timeout 300 python tools/dbg_flow.py 2>&1 | head -20
timeout 900 python -m pytest tests -m gpu -x -q -k "flow or byte_parity or bit_parity or device_errors" > gpurun_out/quick_tests.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/quick_tests.log
timeout 600 python tools/lz_variants.py 2>&1 | tee gpurun_out/lz_variants.log
