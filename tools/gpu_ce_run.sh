cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "not dist" 2>&1 | tail -2
python tools/prof_solve.py --ce --n 1025 2>&1 | tail -2
python tools/prof_solve.py --n 1025 --its 1000 2>&1 | tail -1
python tools/prof_solve.py --n 1025 --its 1000 2>&1 | tail -1
