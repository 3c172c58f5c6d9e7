# dev sweep: staged L2HMC step time vs row-program chunk size / occupancy target
for cc in ${CCS:-1200 2400 4800}; do for mb in ${MBS:-0 4 5 6 8}; do
  echo "cc=$cc mb=$mb $(SF_CHUNK_COST=$cc SF_MIN_BLOCKS=$mb timeout 600 python tools/l2hmc_perf.py 100000 2>&1 | tail -2 | tr '\n' ' ')"
done; done
