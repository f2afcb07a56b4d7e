cd $GRAFT_REPO_ROOT
for i in 1 2; do python tools/time_ops.py 2>&1 | head -1; done
LVL=4 ET=64 python tools/time_ops.py 2>&1 | head -1
python tools/time_kvar.py 2>&1 | tail -1
python -m pytest tests/test_assembly_gpu.py -x -q 2>&1 | tail -3
