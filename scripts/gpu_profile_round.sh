# Refresh the round's bench lines and ncu evidence (profiles/ is filled from gpurun_out/).
mkdir -p gpurun_out/prof
P=gpurun_out/prof
python bench.py --steps 20 --warmup 5 > $P/bench_wan.json 2> $P/bench_wan.err
python bench.py --steps 200 --warmup 5 --no-extra --no-cpu > $P/bench_wan_200.json 2> $P/bench_wan_200.err
python bench.py --workload cog --no-extra > $P/bench_cog.json 2> $P/bench_cog.err
python bench.py --variant asa_gt --no-cpu --no-extra > $P/bench_wan_gt.json 2>&1
python bench.py --tau-mode --no-cpu --no-extra > $P/bench_wan_tau.json 2>&1
python bench.py --impl reference --steps 20 --warmup 5 > $P/bench_ref.json 2>&1
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-extra"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $P/launches_wan.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $P/launches_cog.csv $B --workload cog > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -s 8 -c 5 -o $P/full_wan -f $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -s 8 -c 5 -o $P/full_cog -f $B --workload cog > /dev/null 2>&1
ls -la $P
