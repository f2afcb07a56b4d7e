cd $GRAFT_REPO_ROOT
for env in "X=1" "HB_MOMENT_FROM=0" "HB_MOMENTS=1"; do
  echo "== c3 $env"; env $env python bench.py --config 3 --no-cpu-baseline --steps 2 --warmup 1 2>/dev/null | python -c "
import json,sys
r=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(r['ms_per_step'])"
  echo "== c5 $env"; env $env python bench.py --config 5 --no-cpu-baseline --steps 2 --warmup 1 2>/dev/null | python -c "
import json,sys
r=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(r['ms_per_step'])"
done
