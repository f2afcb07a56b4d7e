cd $GRAFT_REPO_ROOT
for i in 1 2; do python tools/time_ops.py 2>&1 | head -1; HB_LIB_PATH=variants_tmp/old/libheatbem_b200.so python tools/time_ops.py 2>&1 | head -1; done
python tools/hash_ops.py > gpurun_out/hash_new.txt 2>&1
HB_LIB_PATH=variants_tmp/old/libheatbem_b200.so python tools/hash_ops.py > gpurun_out/hash_old.txt 2>&1
diff gpurun_out/hash_new.txt gpurun_out/hash_old.txt && echo "hashes identical"
