mkdir -p gpurun_out/r02e22
P=gpurun_out/r02e22
timeout 1500 python -m pytest tests -m gpu -q -x > $P/pytest_gpu.log 2>&1; echo "rc=$?" >> $P/pytest_gpu.log
tail -2 $P/pytest_gpu.log
python bench.py --workload cog --no-extra --no-cpu > $P/bench_cog.json 2> $P/bench_cog.err
python bench.py --steps 20 --warmup 5 --no-cpu > $P/bench_wan.json 2> $P/bench_wan.err
python3 -c "
import json
for f in ['$P/bench_cog.json','$P/bench_wan.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d['ms_per_step'], d['ms_attn'], d['roofline']['frac'], d['clocks'])
    if d.get('cog'): print('  cog', d['cog']['ms_per_step'], d['cog']['ms_attn'])
"
