python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for A in 1 8 1 8; do for c in C2_2d_101x101_Nv32 C3_2d_141x141_jitter_Nv32; do BGK_NCS2_ALIGN=$A timeout 300 python tools/phase_times.py --config $c --steps 20 --warmup 3 2>&1 | tail -1; done; done
