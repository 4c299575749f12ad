# decoder change check: parity subset + C2 decode/lz77 times + whole-file configs
timeout 900 python -m pytest tests -m gpu -x -q -k "bit or decoder or warp_spec or split or code_length or full_size or errors" > gpurun_out/dec_tests.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/dec_tests.log
timeout 300 python tools/time_phase.py decode; timeout 300 python tools/time_phase.py lz77; timeout 300 python tools/time_phase.py all
timeout 600 python tools/lz_whole.py C2,C5,C2-S16
