cd $GRAFT_REPO_ROOT
run() { name=$1; shift; bash tools/build_variant.sh $name "$@" > /dev/null 2>gpurun_out/var_$name.err || { echo "build $name failed"; return; }; echo "== $name $@"; HB_LIB_PATH=variants_tmp/$name/libheatbem_b200.so python tools/time_ops.py 2>&1 | head -1; }
run base
run w10 -DHB_PAIR_WARPS=10
run w12 -DHB_PAIR_WARPS=12
run w6m3 -DHB_PAIR_WARPS=6 -DHB_PAIR_MINB=3
run q4 -DHB_QGROUP=4
run q1 -DHB_QGROUP=1
run w16m1 -DHB_PAIR_WARPS=16 -DHB_PAIR_MINB=1
