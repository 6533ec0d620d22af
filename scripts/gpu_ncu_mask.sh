set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine_kernel -s 2 -c 1 -o gpurun_out/refine_keep51 -f $B > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine_kernel -s 2 -c 1 -o gpurun_out/refine_tau095 -f $B --tau-mode --tau 0.95 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:probe_tc_kernel -s 2 -c 1 -o gpurun_out/probe_wan -f $B > gpurun_out/ncu3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_tc_kernel -s 2 -c 1 -o gpurun_out/attn_cog -f $B --workload cog > gpurun_out/ncu4.log 2>&1
ls -la gpurun_out
