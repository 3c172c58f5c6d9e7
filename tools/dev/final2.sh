python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r02p.txt 2>&1; tail -2 gpurun_out/gputests_r02p.txt
python bench.py > gpurun_out/bench_r02p.json 2> gpurun_out/bench_r02p.err
python bench.py --impl reference > gpurun_out/bench_ref_r02p.json 2> gpurun_out/bench_ref_r02p.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l2hmc_launches_r02p.csv python tools/l2hmc_steps.py 100000 5 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sf_rows -s 3 -c 1 -f -o gpurun_out/rows_r02p python tools/l2hmc_steps.py 100000 5 > /dev/null 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/resnet_launches_r02p.csv python tools/resnet_step.py 32 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sf_uni --csv --log-file gpurun_out/c2_launches_r02p.csv python tools/c2_profile.py > /dev/null 2>&1
echo done
