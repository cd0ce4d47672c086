#!/bin/bash
# tools/ab_varlen.sh lib1.so lib2.so ... : per-variant hash_varlen call times on
# config 2 and the bench's config-2 step (4 variants, one CUDA graph) per library
for r in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = default ]; then unset HTH_LIB; else export HTH_LIB=$lib; fi
    python tools/exp_varlen.py 2>&1 | tail -4 | tr '\n' ' ' | sed 's/  */ /g'; echo
    python bench.py --workload cfg2 --steps 30 --warmup 5 --no-extra --e2e-steps 0 --no-check 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('   $lib cfg2 step', round(d['ms_per_step']*1e3,1), 'us', round(d['value']), 'GB/s')"
  done
done
