cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "not dist" 2>&1 | tail -2
for m in 1 0; do echo "cfg2 march=$m: $(HADR_STENCIL_MARCH=$m python tools/prof_solve.py --n 1025 --its 1000 2>&1 | tail -1)"; done
for m in 1 0; do echo "cfg4 513 march=$m: $(HADR_STENCIL_MARCH=$m HADR_WORKLOAD=cfg4 python tools/prof_solve.py --n 513 --its 1000 2>&1 | tail -1)"; done
for m in 1 0; do echo "cfg3 2049 march=$m: $(HADR_STENCIL_MARCH=$m HADR_WORKLOAD=cfg3 python tools/prof_solve.py --n 2049 --its 1000 2>&1 | tail -1)"; done
python - <<'PY'
import sys; sys.path.insert(0,'tools'); sys.path.insert(0,'.')
from k1_kernel import k1_measure
from paper_1712_06091_b200 import workloads, _lib
wl = workloads.cfg2(1025)
for m in (1, 0):
    _lib.set_option("stencil_march", m)
    for v in (0, 1):
        r = k1_measure(wl, reps=50, variant=v)
        print("march", m, "variant", v, {k: r[k] for k in r if 'ms' in k or 'GB' in k})
PY
