# Interleaved A/B of the mask time (ms_mask) and fused step for library variants:
# ab_mask.sh "<workloads>" lib1 lib2 ...
for rep in 1 2 3; do
  for lib in "${@:2}"; do
    for wl in $1; do
      BLADE_LIB=$lib python bench.py --no-cpu --no-e2e --steps 100 --workload $wl \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$rep $lib $wl mask', round(d['ms_mask'],4), 'fused', round(d['ms_per_step'],4))"
    done
  done
done
