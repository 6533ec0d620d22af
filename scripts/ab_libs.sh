# A/B timing of attention library variants: ab_libs.sh "<wl:attn> ..." lib1 lib2 ...
# prints ms_attn per (lib, workload) for two interleaved rounds.
cfgs="$1"; shift
for rep in 1 2; do
  for lib in "$@"; do
    for c in $cfgs; do
      wl=${c%%:*}; at=${c##*:}
      BLADE_LIB=$lib python bench.py --no-cpu --no-e2e --steps 100 --workload $wl --attn $at \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rep $lib $wl $at', round(d['ms_attn'],4), d['clocks']['sm_mhz'])"
    done
  done
done
