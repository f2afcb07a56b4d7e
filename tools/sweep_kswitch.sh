#!/usr/bin/env bash
# K direct / moment switch block at config 5 (HB_K_MOMENT_FROM): bench --config 5 step time per setting
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for k in 62 32 92 122; do
  echo "== HB_K_MOMENT_FROM=$k"; HB_K_MOMENT_FROM=$k python bench.py --config 5 --no-cpu-baseline --steps 2 --warmup 1 2>/dev/null | python -c "
import json,sys
r=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(r['ms_per_step'])"
done
