mkdir -p gpurun_out
RSGRAD_BSLICE_NW=4 timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bslice" 2>&1 | tail -1
for nw in 8 4; do echo nw=$nw; RSGRAD_BSLICE_NW=$nw python scripts/bench_layer.py 64 10 bslice_bwd; RSGRAD_BSLICE_NW=$nw python scripts/bench_paper.py g16x16; done
