for v in "SF_ROW_CTA_CHAINS=256" "SF_ROW_LOOPSYNC=1 SF_ROW_CTA_CHAINS=256" "SF_ROW_LOOPSYNC=1 SF_ROW_CTA_CHAINS=512" "SF_ROW_LOOPSYNC=1 SF_ROW_CTA_CHAINS=704" "SF_ROW_LOOPSYNC=1 SF_ROW_REPLICAS=2 SF_ROW_CTA_CHAINS=128" "SF_ROW_LOOPSYNC=1 SF_ROW_REPLICAS=2 SF_ROW_CTA_CHAINS=384"; do env $v python tools/l2hmc_event_time.py 100000; done
M="--section SpeedOfLight --section SchedulerStats --section WarpStateStats --section Occupancy --section LaunchStats --section InstructionStats"
for v in "SF_ROW_REPLICAS=2 SF_ROW_GRID=legacy" "SF_ROW_CTA_CHAINS=256"; do
  env $v ncu $M --clock-control none -k regex:sf_rows -s 3 -c 1 python tools/l2hmc_steps.py 100000 5 > gpurun_out/exp5_$(echo $v | tr ' =' '__').txt 2>&1
done
