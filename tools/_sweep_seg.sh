cd $GRAFT_REPO_ROOT
for s in 4 16 32 64; do echo "== c2 ipw $s"; HB_ITEMS_PER_WARP=$s python tools/time_ops.py 2>&1 | head -1; done
for s in 4 16 64 256; do echo "== c2 ipw_m $s"; HB_ITEMS_PER_WARP_M=$s python tools/time_ops.py 2>&1 | head -1; done
for s in 32 16 8; do echo "== L4 E64 seg $s"; HB_ITEMS_PER_WARP=1 HB_SEG_LEN=$s LVL=4 ET=64 python tools/time_ops.py 2>&1 | head -1; done
for s in 32 8; do echo "== L2 E32 seg $s"; HB_ITEMS_PER_WARP=1 HB_SEG_LEN=$s LVL=2 ET=32 python tools/time_ops.py 2>&1 | head -1; done
