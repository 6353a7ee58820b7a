for W in 2 4 2 4; do BGK_TRANSPORT_WPB=$W timeout 300 python tools/phase_times.py --steps 5 --warmup 2 2>&1 | tail -1; done
