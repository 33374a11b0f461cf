#!/bin/bash
# Round profiling on the GPU box: bench line, ncu launch list of the bench command, and one
# ncu --set full capture per ICP kernel (C4, certified run) -> gpurun_out/
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/ncu_cert.py 42 > gpurun_out/ncu_pre.log 2>&1
for spec in "icp_nn:3:nn_it3" "icp_nn:41:nn_it41" "icp_select:41:sel_it41" "icp_acc:41:acc_it41"; do
  IFS=: read k s name <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o gpurun_out/prof_$name -f python tools/ncu_cert.py 42 > gpurun_out/ncu_$name.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:icp_proj -s 10 -c 1 \
    -o gpurun_out/prof_proj_c3 -f python tools/ncu_proj.py > gpurun_out/ncu_proj_c3.log 2>&1
timeout 900 python tools/bench_all.py 5 > gpurun_out/bench_all.jsonl 2> gpurun_out/bench_all.err
python tools/probe_stamps.py c4 > gpurun_out/stamps.log 2>&1
ls -la gpurun_out
