python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
python -m pytest tests -m gpu -x -q > gpurun_out/gputests_r02q.txt 2>&1; tail -2 gpurun_out/gputests_r02q.txt
python bench.py > gpurun_out/bench_r02q.json 2> gpurun_out/bench_r02q.err
python bench.py --impl reference > gpurun_out/bench_ref_r02q.json 2> gpurun_out/bench_ref_r02q.err
echo done
