# ncu --set full of the C2 nn_query kernel and of a warm C4 icp_nn kernel (1 launch each)
set -e
python tools/ncu_nn.py > gpurun_out/p1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:nn_query_kernel -s 1 -c 1 -o gpurun_out/prof_c2 -f python tools/ncu_nn.py > gpurun_out/ncu1.log 2>&1
python tools/ncu_run.py point_to_plane 12 > gpurun_out/p2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:icp_nn -s 10 -c 1 -o gpurun_out/prof_nn2 -f python tools/ncu_run.py point_to_plane 12 > gpurun_out/ncu2.log 2>&1
