cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "rc=$?"
tail -3 gpurun_out/bench_full.err
python tools/prof_solve.py --n 1025 --its 3 > gpurun_out/pl.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/prof_solve.py --n 1025 --its 3 > gpurun_out/ncu_l.log 2>&1; echo "ncu rc=$?"
