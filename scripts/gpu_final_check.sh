# Full GPU validation + refreshed evidence for profiles/ (run near the end of a round;
# then `python scripts/collect_profiles.py rNN` here).
mkdir -p gpurun_out/prof
P=gpurun_out/prof
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $P/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tests/tools/sanitize_cases.py > $P/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> $P/sanitizer_$tool.log
done
bash scripts/gpu_profile_round.sh
python scripts/mask_time.py --workload wan > $P/mask_time_wan.jsonl 2>&1
python scripts/mask_time.py --workload cog --configs keep25,tau0.9,tau0.95 > $P/mask_time_cog.jsonl 2>&1
python scripts/sweep.py --steps 10 > $P/sweep_wan.jsonl 2>/dev/null
# pipe counters (tensor / XU=MUFU / shared / FMA / fp64 / DMMA) of every kernel of a step
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extra"
ncu --metrics $M --clock-control none -s 10 -c 12 --csv --log-file $P/pipes_wan.csv $B > /dev/null 2>&1
ncu --metrics $M --clock-control none -s 10 -c 12 --csv --log-file $P/pipes_cog.csv $B --workload cog > /dev/null 2>&1
ncu --metrics $M --clock-control none -s 10 -c 12 --csv --log-file $P/pipes_wan_tau95.csv $B --tau-mode --tau 0.95 > /dev/null 2>&1
python scripts/bench_bwd.py > $P/bench_bwd_wan.json 2>&1
python scripts/bench_bwd.py --workload cog > $P/bench_bwd_cog.json 2>&1
python scripts/bench_bwd.py --variant asa_gt > $P/bench_bwd_wan_asa_gt.json 2>&1
python scripts/bench_bwd.py --workload cog --variant asa_gt > $P/bench_bwd_cog_asa_gt.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bwd -c 8 --csv --log-file $P/launches_bwd_wan.csv python scripts/bench_bwd.py --steps 1 > /dev/null 2>&1
cat $P/pytest_gpu.log $P/smoke.log
ls -la $P
