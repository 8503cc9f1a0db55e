cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for p in 1 0 1 0; do echo "pdl=$p: $(HADR_PDL=$p python tools/prof_solve.py --n 1025 --its 1000 2>&1 | tail -1)"; done
for p in 1 0; do echo "cfg4 257 pdl=$p: $(HADR_PDL=$p HADR_WORKLOAD=cfg4 python tools/prof_solve.py --n 257 --its 1000 2>&1 | tail -1)"; done
for p in 1 0; do echo "cfg3 1025 pdl=$p: $(HADR_PDL=$p HADR_WORKLOAD=cfg3 python tools/prof_solve.py --n 1025 --its 1000 2>&1 | tail -1)"; done
