# round-2 profiles: launch list of the bench command, full captures of the TC kernels
# (L2 flushed before each kernel = ncu default, and --cache-control none = warm, as back
# to back), the d16 CUDA-core backward and the mixer
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extra"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_launches.csv $B > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:swr_tc_kernel -s 6 -c 2 -o gpurun_out/r02_tc_full $B > gpurun_out/ncu_tc.log 2>&1; echo "tc full rc=$?"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:swr_tc_kernel -s 6 -c 2 -o gpurun_out/r02_tc_warm $B > gpurun_out/ncu_tcw.log 2>&1; echo "tc warm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:swr_tc_kernel -s 6 -c 2 -o gpurun_out/r02_mix_full $B --op mix > gpurun_out/ncu_mix.log 2>&1; echo "mix full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_stream|bwd_ffma_vec" -s 6 -c 2 -o gpurun_out/r02_d16_full $B --config paper_d16 > gpurun_out/ncu_d16.log 2>&1; echo "d16 full rc=$?"
