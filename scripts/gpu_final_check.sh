# Full GPU validation + refreshed evidence for profiles/ (run near the end of a round).
mkdir -p gpurun_out/prof
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/prof/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/prof/smoke.log 2>&1
bash scripts/gpu_profile_round.sh
python scripts/bench_bwd.py > gpurun_out/prof/bench_bwd_wan.json 2>&1
python scripts/bench_bwd.py --workload cog > gpurun_out/prof/bench_bwd_cog.json 2>&1
python scripts/bench_bwd.py --variant asa_gt > gpurun_out/prof/bench_bwd_wan_asa_gt.json 2>&1
python scripts/bench_bwd.py --workload cog --variant asa_gt > gpurun_out/prof/bench_bwd_cog_asa_gt.json 2>&1
python scripts/sweep.py --steps 10 > gpurun_out/prof/sweep_wan.jsonl 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bwd -c 8 --csv --log-file gpurun_out/prof/launches_bwd_wan.csv python scripts/bench_bwd.py --steps 1 > /dev/null 2>&1
for wl in wan cog; do ncu --set full --import-source on --clock-control none -k regex:_tc_kernel -s 2 -c 2 -o gpurun_out/prof/full_bwd_$wl -f python scripts/bench_bwd.py --workload $wl --steps 1 > /dev/null 2>&1; done
cat gpurun_out/prof/pytest_gpu.log gpurun_out/prof/smoke.log
