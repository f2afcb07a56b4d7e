cd $GRAFT_REPO_ROOT
for ng in 0 1; do echo "== HB_FIN_NODE_GRID=$ng"; HB_FIN_NODE_GRID=$ng python tools/time_ops.py 2>&1 | head -1; HB_FIN_NODE_GRID=$ng LVL=4 ET=64 python tools/time_ops.py 2>&1 | head -1; HB_FIN_NODE_GRID=$ng python tools/hash_ops.py > gpurun_out/hash_ng$ng.txt 2>&1; done
diff gpurun_out/hash_ng0.txt gpurun_out/hash_ng1.txt && echo "hashes identical"
