# Interleaved A/B of attention impls on one library: ab_attn.sh "<wl:attn> ..." [reps]
for rep in $(seq 1 ${2:-3}); do
  for c in $1; do
    wl=${c%%:*}; at=${c##*:}
    python bench.py --no-cpu --no-e2e --steps 100 --workload $wl --attn $at \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rep $wl $at fused', round(d['ms_per_step'],4), 'attn', round(d['ms_attn'],4), 'mask', round(d['ms_mask'],4), d['clocks']['sm_mhz'])"
  done
done
