cd $GRAFT_REPO_ROOT
for db in 0 1; do echo "== c2 HB_CURL_DB=$db"; HB_CURL_DB=$db python tools/time_ops.py 2>&1 | tail -1; HB_CURL_DB=$db LVL=4 ET=64 python tools/time_ops.py 2>&1 | tail -1; done
for db in 0 1; do echo "== c5 chunk HB_CURL_DB=$db"; HB_CURL_DB=$db python tools/prof_c5_d.py 2>&1 | tail -1; done
python -m pytest tests/test_assembly_gpu.py -x -q -k "curl or hypersingular or D_ or c1 or c2" 2>&1 | tail -3
