# sparsity sweep (BJ configs[3]) and ASA_GT backward with the round-2 kernels
mkdir -p gpurun_out/r02sw
P=gpurun_out/r02sw
timeout 900 python scripts/sweep.py > $P/sweep_wan.jsonl 2> $P/sweep_wan.err
timeout 600 python scripts/sweep.py --workload cog > $P/sweep_cog.jsonl 2> $P/sweep_cog.err
python scripts/bench_bwd.py --variant asa_gt > $P/bench_bwd_wan_asa_gt.json 2>&1
python scripts/bench_bwd.py --workload cog --variant asa_gt > $P/bench_bwd_cog_asa_gt.json 2>&1
wc -l $P/*.jsonl; tail -2 $P/bench_bwd_*
