for c in 160 192 224 256 288 320 384 448 512; do SF_ROW_CTA_CHAINS=$c python tools/l2hmc_event_time.py 10000 100000; done
for c in 256 320 512; do SF_ROW_GRID=legacy SF_ROW_CTA_CHAINS=$c python tools/l2hmc_event_time.py 100000; done
SF_ROW_CTA_CHAINS=256 python tools/l2hmc_event_time.py 100000
SF_ROW_CTA_CHAINS=256 python tools/l2hmc_event_time.py 100000
python tools/l2hmc_event_time.py 100000
