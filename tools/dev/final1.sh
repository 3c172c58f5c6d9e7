python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r02o.txt 2>&1; tail -2 gpurun_out/gputests_r02o.txt
python bench.py > gpurun_out/bench_r02o.json 2> gpurun_out/bench_r02o.err
python bench.py --impl reference > gpurun_out/bench_ref_r02o.json 2> gpurun_out/bench_ref_r02o.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/bench_launches_r02o.csv python bench.py --steps 2 --warmup 3 --quick > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sf_rows -s 3 -c 1 -f -o gpurun_out/rows_r02o python tools/l2hmc_steps.py 100000 5 > gpurun_out/ncu_rows.log 2>&1
echo done
