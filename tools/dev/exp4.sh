SF_ROW_CTA_CHAINS=256 python tools/l2hmc_event_time.py 10000 100000
for c in 64 128 192 256; do SF_ROW_REPLICAS=2 SF_ROW_CTA_CHAINS=$c python tools/l2hmc_event_time.py 10000 100000; done
SF_ROW_REPLICAS=2 SF_ROW_GRID=legacy python tools/l2hmc_event_time.py 100000
SF_ROW_REPLICAS=2 python -m pytest -q -x tests/test_gpu_l2hmc_headline.py tests/test_gpu_workloads.py 2>&1 | tail -3
