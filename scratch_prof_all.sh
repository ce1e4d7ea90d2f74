set -x
# host-driven loop (same kernels as the sweep graph; ncu cannot attribute kernels inside conditional graph bodies)
STMF_GRAPH=0 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_c2_launches.csv python scratch_launch.py 2 4 > gpurun_out/p_c2.log 2>&1
STMF_GRAPH=0 ncu --set full --import-source on --clock-control none -k regex:k_phaseB --launch-skip 300 --launch-count 1 -o gpurun_out/p_c2_phaseB python scratch_prof.py 2 1.5 1 > gpurun_out/p_c2b.log 2>&1
ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p_c2_graph.csv python scratch_time.py 2 3 > gpurun_out/p_c2g.log 2>&1
STMF_GRAPH=0 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p_c3_launches.csv python scratch_launch.py 3 0 4 > gpurun_out/p_c3.log 2>&1
echo done
