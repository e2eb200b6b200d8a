timeout 300 python tools/batch_probe.py 16x32i 16x32 16x64i 16x256 16x1024 8x16384i 8x65536 8x262144
