#!/bin/bash
# Row-kernel launch-geometry sweep behind DESIGN.md §4 (round 2): device time
# per staged L2HMC transition (warm, and with the bench's 256 MiB L2 flush)
# for the grid / CTA size / loop-barrier / two-chains-per-thread variants.
#   gpurun -- bash tools/row_grid_sweep.sh
set -u
B="10000 100000"
run() { env "$@" FLUSH=1 python tools/l2hmc_event_time.py $B; }
run SF_ROW_GRID=legacy SF_ROW_LOOPSYNC=0                  # 128-chain CTAs (round-2 first half)
run SF_ROW_LOOPSYNC=0 SF_ROW_CTA_THREADS=256              # balanced, 256-thread CTAs
run SF_ROW_LOOPSYNC=0                                     # balanced, one 704-thread CTA per SM
run SF_ROW_LOOPSYNC=1                                     # + a barrier per loop iteration (default)
run SF_ROW_LOOPSYNC=1 SF_ROW_SYNC_EVERY=300               # + barriers in straight-line code
run SF_ROW_REPLICAS=2                                     # two chains per thread, FFMA2 immediates
run SF_TEAM_MAX_BATCH=1000000000                          # team split at every batch
