R=r2
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/${R}_launches_bench_c4.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-iter-profile > gpurun_out/${R}_ncu_bench.log 2>&1
timeout 900 python tools/bench_all.py 5 > gpurun_out/${R}_bench_all.jsonl 2> gpurun_out/${R}_bench_all.err
python tools/probe_stamps.py c4 > gpurun_out/${R}_stamps.log 2>&1
python tools/time_small.py > gpurun_out/${R}_time_small.log 2>&1
ls -la gpurun_out | tail -8
cut -c1-250 gpurun_out/${R}_bench.json
