#!/bin/bash
# A/B of library variants on c2: setup_ms / loop_ms / ms_per_step per variant.
for lib in paper_1502_01645_b200/lib/libalnnls.so "$@"; do
  ALNNLS_LIB=$lib python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('%-40s setup %.3f loop %.3f step %.3f' % ('$lib', d['setup_ms'], d['loop_ms'], d['ms_per_step']))"
done
