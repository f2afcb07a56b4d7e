import sys, os, numpy as np
R=os.environ.get("GRAFT_REPO_ROOT","/root/repo"); sys.path.insert(0,R); sys.path.insert(0,R+"/tests")
import paper_2102_09811_b200 as hb
from oracle import oracle as O
from _hb_util import rel_block_err
O.build()
m = hb.generate_cube_surface(2); tg = hb.TimeGrid(1.0, 80); p = hb.KernelParams(0.5, tg.step, length_scale=m.diameter)
Q4=hb.QuadratureConfig()
F={"V": lambda: hb.assemble_single_layer(m,tg,p,Q4), "K": lambda: hb.assemble_double_layer(m,tg,p,Q4), "D2": lambda: hb.assemble_hypersingular_d2(m,tg,p,Q4)}
for op,f in F.items():
    ref=O.assemble(m,tg,p,Q4,op); x=O.assemble(m,tg,p,Q4,op,exact=True); got=f().blocks
    e=rel_block_err(ref,x); a=rel_block_err(got,x)
    bad=np.flatnonzero(a > e + 1e-13)
    print(op, "max ratio %.2f"%np.max(a/e), "bad d", bad[:20], "ratios", np.round((a/e)[bad[:10]],2), "eps", e[bad[:5]])
