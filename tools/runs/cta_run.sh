BGK_TRANSPORT_R=13 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cta_shared" 2>&1 | tail -3
for G in 8 4; do BGK_TRANSPORT_R=13 BGK_TRANSPORT_CTA=$G timeout 300 python tools/phase_times.py --steps 3 --warmup 2 2>&1 | tail -1; done
BGK_TRANSPORT_R=13 timeout 300 python tools/phase_times.py --steps 3 --warmup 2 2>&1 | tail -1
