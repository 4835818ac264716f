#!/bin/bash
# lean (1 target / thread) vs dense (2-target units, padded pairs, row items) across D_occ 2..6
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
C=${C:-lowd2_1e7,lowd3_1e7,lowd4_1e7,lowd6_1e7}
timeout 900 python tools/sweep.py --configs $C --tpi 1 --ns 1 --nbuf 1 --nt 64 --pad 0 --reps 9 2>&1 | grep -v Warn
timeout 900 python tools/sweep.py --configs $C --tpi 1 --ns 3 --nbuf 1 --nt 64 --pad 0 --reps 9 2>&1 | grep -v Warn
timeout 900 python tools/sweep.py --configs $C --tpi 2 --ns 3 --nbuf 1 --nt 128,64 --pad 1 --reps 9 2>&1 | grep -v Warn
timeout 900 python tools/sweep.py --configs $C --tpi 2 --ns 3 --nbuf 1 --nt 128 --pad 1 --tile 2 --reps 9 2>&1 | grep -v Warn
