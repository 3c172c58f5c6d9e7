for e in 0 150 300 600; do
for v in "SF_ROW_CTA_CHAINS=704" "SF_ROW_REPLICAS=2 SF_ROW_CTA_CHAINS=384" "SF_ROW_REPLICAS=2 SF_ROW_CTA_CHAINS=192"; do env SF_ROW_LOOPSYNC=1 SF_ROW_SYNC_EVERY=$e $v python tools/l2hmc_event_time.py 100000 | cut -c1-150; done; done
