set -x
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 800 --csv --log-file gpurun_out/launches_c3_r2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/profile_net.py --net sd15 > gpurun_out/plain_pn.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:attn_tc_kernel -c 2 -o gpurun_out/r2_attn_sd15 python tools/profile_net.py --net sd15 > gpurun_out/ncu_attn.log 2>&1
python tools/profile_net.py --net dit > gpurun_out/plain_pn2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:gemm -c 8 -o gpurun_out/r2_gemm_dit python tools/profile_net.py --net dit > gpurun_out/ncu_dit.log 2>&1
python tools/gemm_traffic.py record --net sd15 > gpurun_out/gemm_algo.json 2> gpurun_out/gemm_algo.err && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none --profile-from-start off -k regex:gemm --csv --log-file gpurun_out/gemm_dram.csv python tools/profile_net.py --net sd15 > gpurun_out/ncu_dram.log 2>&1
ls -la gpurun_out | tail -20
