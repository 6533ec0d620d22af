# Refresh the round's bench lines and ncu evidence (profiles/ is filled from gpurun_out/).
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/bench_wan.json 2> gpurun_out/prof/bench_wan.err
python bench.py --workload cog > gpurun_out/prof/bench_cog.json 2> gpurun_out/prof/bench_cog.err
python bench.py --variant asa_gt --no-cpu > gpurun_out/prof/bench_wan_gt.json 2>&1
python bench.py --impl reference --steps 3 --warmup 0 > gpurun_out/prof/bench_ref.json 2>&1
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/prof/launches_wan.csv $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/prof/launches_cog.csv $B --workload cog > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -s 8 -c 5 -o gpurun_out/prof/full_wan -f $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -s 8 -c 5 -o gpurun_out/prof/full_cog -f $B --workload cog > /dev/null 2>&1
ls -la gpurun_out/prof
