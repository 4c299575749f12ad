for i in 1 2 3; do timeout 600 python tools/decode_time.py 148,296,1024; done
