# End-of-round evidence on one B200 (product build): GPU suite, smoke, bench lines, mask and
# backward timings, sparsity sweep, launch lists, pipe counters, ncu full captures.
#   gpurun --timeout 3000 -- 'bash scripts/gpu_round_evidence.sh [outdir]'
P=${1:-gpurun_out/evidence}
mkdir -p $P
python -c "import __graft_entry__ as g; g.build()" > $P/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $P/pytest_gpu.log 2>&1; echo "rc=$?" >> $P/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $P/smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > $P/bench_wan.json 2> $P/bench_wan.err
python bench.py --impl reference --steps 20 --warmup 5 > $P/bench_ref.json 2> $P/bench_ref.err
python bench.py --workload cog --no-extra --no-cpu > $P/bench_cog.json 2> $P/bench_cog.err
python bench.py --tau-mode --no-extra --no-cpu > $P/bench_wan_tau.json 2> $P/bench_wan_tau.err
python bench.py --variant asa_gt --no-extra --no-cpu > $P/bench_wan_gt.json 2> $P/bench_wan_gt.err
python scripts/mask_time.py --workload wan > $P/mask_time_wan.jsonl 2>&1
python scripts/mask_time.py --workload cog --configs keep25,tau0.9,tau0.95 > $P/mask_time_cog.jsonl 2>&1
python scripts/bench_bwd.py > $P/bench_bwd_wan.json 2>&1
python scripts/bench_bwd.py --workload cog > $P/bench_bwd_cog.json 2>&1
python scripts/bench_bwd.py --variant asa_gt > $P/bench_bwd_wan_asa_gt.json 2>&1
python scripts/bench_bwd.py --workload cog --variant asa_gt > $P/bench_bwd_cog_asa_gt.json 2>&1
timeout 900 python scripts/sweep.py > $P/sweep_wan.jsonl 2> $P/sweep_wan.err
timeout 600 python scripts/sweep.py --workload cog > $P/sweep_cog.jsonl 2> $P/sweep_cog.err
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $P/launches_wan.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $P/launches_cog.csv $B --workload cog > /dev/null 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_active.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum
ncu --metrics $M --clock-control none -s 10 -c 12 --csv --log-file $P/pipes_wan.csv $B > /dev/null 2>&1
ncu --metrics $M --clock-control none -s 10 -c 12 --csv --log-file $P/pipes_cog.csv $B --workload cog > /dev/null 2>&1
ncu --metrics $M --clock-control none -s 12 -c 12 --csv --log-file $P/pipes_wan_tau95.csv $B --tau-mode --tau 0.95 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_tc2p -s 2 -c 1 -o $P/full_wan_attn -f $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_tc2p -s 2 -c 1 -o $P/full_cog_attn -f $B --workload cog > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:probe2 -s 2 -c 1 -o $P/full_wan_probe -f $B > /dev/null 2>&1
tail -3 $P/pytest_gpu.log; cat $P/smoke.log; ls -la $P
