M="--section SpeedOfLight --section SchedulerStats --section WarpStateStats --section Occupancy --section LaunchStats --metrics sm__cycles_active.avg,sm__cycles_active.max,sm__cycles_active.min,sm__cycles_elapsed.max,smsp__inst_executed.sum,sm__ctas_launched.max,sm__ctas_launched.min,sm__warps_launched.max,sm__warps_launched.min,smsp__warps_launched.max,smsp__warps_launched.min"
for v in "SF_ROW_GRID=legacy" "SF_ROW_GRID=legacy SF_ROW_CTA_CHAINS=256" "SF_ROW_CTA_CHAINS=160" "SF_ROW_CTA_CHAINS=256"; do
  env $v ncu $M --clock-control none -k regex:sf_rows -s 3 -c 1 python tools/l2hmc_steps.py 100000 5 > gpurun_out/exp3_$(echo $v | tr ' =' '__').txt 2>&1
done
