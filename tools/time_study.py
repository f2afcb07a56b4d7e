"""Time the study driver (run_level, GPU backend) at levels 0..L of the
default Dirichlet study (heatbem/study.py defaults)."""
import json, os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2102_09811_b200 as hb

L = int(os.environ.get("LEVELS", "3"))
hb.run_level(hb.StudyConfig(), 0)   # warm-up (library load, tables)
out = []
for lv in range(L):
    t0 = time.perf_counter()
    r = hb.run_level(hb.StudyConfig(), lv)
    out.append({"level": lv, "E_t": r.E_t, "E_x": r.E_x, "s": round(time.perf_counter() - t0, 3),
                "err_computed": r.err_computed, "err_repr": r.err_repr, "iterations": r.iterations,
                "timings": r.seconds_assembly})
print(json.dumps(out))
print(hb.results_to_csv([hb.LevelResult(**{k: o[k] for k in ("level", "E_t", "E_x", "err_computed")},
                                        err_projected=float("nan"), err_repr=o["err_repr"], iterations=o["iterations"],
                                        residual=0.0, converged=True) for o in out]))
