set -x
B="200 2000 10000 100000"
SF_ROW_GRID=legacy python tools/l2hmc_event_time.py $B
python tools/l2hmc_event_time.py $B
SF_ROW_CTA_CHAINS=256 python tools/l2hmc_event_time.py $B
SF_ROW_CTA_CHAINS=704 python tools/l2hmc_event_time.py 100000
SF_TEAM_MAX_BATCH=1000000000 python tools/l2hmc_event_time.py 10000 100000
SF_TEAM_MAX_BATCH=1000000000 SF_ROW_CTA_CHAINS=256 python tools/l2hmc_event_time.py 10000 100000
SF_ROW_GRID=legacy SF_TEAM_MAX_BATCH=1000000000 python tools/l2hmc_event_time.py 10000 100000
python -m pytest -q -x tests/test_gpu_l2hmc_headline.py tests/test_gpu_workloads.py 2>&1 | tail -3
