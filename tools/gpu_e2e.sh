for st in 2 3 4; do for mb in 48 128; do SPN_HOST_STREAMS=$st SPN_HOST_CHUNK_MB=$mb timeout 300 python tools/e2e_probe2.py; done; done
