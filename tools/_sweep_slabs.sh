cd $GRAFT_REPO_ROOT
for s in 2 4 6 8 "0.05,0.95" "0.05,0.45,0.5" "0.04,0.16,0.4,0.4" "0.03,0.1,0.27,0.3,0.3" "0.1,0.3,0.3,0.3" "0.02,0.08,0.2,0.35,0.35"; do
  echo "== $s"; HB_E2E_SLABS="$s" python tools/e2e_timeline.py 2>&1 | head -1 | python -c "
import json,sys
r=json.loads(sys.stdin.readline()); t=r['timeline_ms']; import statistics as st
print({k: round(st.median(x[k] for x in t),3) for k in t[0]})"
done
