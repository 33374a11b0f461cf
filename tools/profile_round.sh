#!/bin/bash
# Round profiling on the GPU box -> gpurun_out/ (then copy the summaries into profiles/):
# bench line, ncu launch list of the bench command, one ncu --set full capture per ICP kernel
# of the timed build (C4 certified run, library-default leaf size), the C2 grid query and the
# C1 small-problem run.  R = round tag (default r2).
R=${R:-r2}
set -x
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/${R}_launches_bench_c4.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-iter-profile > gpurun_out/${R}_ncu_bench.log 2>&1
for spec in "icp_nn:3:nn_it3" "icp_nn:41:nn_it41" "icp_select:41:sel_it41" "icp_select:22:sel_it22" "icp_acc:41:acc_it41"; do
  IFS=: read k s name <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 \
      -o gpurun_out/${R}_prof_$name -f python tools/ncu_cert.py 42 > gpurun_out/${R}_ncu_$name.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grid_query -s 2 -c 1 \
    -o gpurun_out/${R}_prof_grid_c2 -f python tools/ncu_c2.py grid > gpurun_out/${R}_ncu_grid_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:icp_small_run -c 1 \
    -o gpurun_out/${R}_prof_small_c1 -f python tools/time_c1.py > gpurun_out/${R}_ncu_small_c1.log 2>&1
timeout 900 python tools/bench_all.py 5 > gpurun_out/${R}_bench_all.jsonl 2> gpurun_out/${R}_bench_all.err
python tools/probe_stamps.py c4 > gpurun_out/${R}_stamps.log 2>&1
ls -la gpurun_out
