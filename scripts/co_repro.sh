cd $GRAFT_REPO_ROOT
MAMG_COARSEST=1 MAMG_NO_PDL=1 TAG=co_nopdl REPS=2 python scripts/time_setup.py 2>&1 | tail -1
MAMG_COARSEST=1 TAG=co SPEC=randk3d:100,100,100,0 REPS=2 python scripts/time_setup.py 2>&1 | tail -1
MAMG_COARSEST=1 TAG=co SPEC=randk3d:120,120,120,0 REPS=2 python scripts/time_setup.py 2>&1 | tail -1
MAMG_COARSEST=1 MAMG_NO_PDL=1 timeout 600 compute-sanitizer --print-limit 5 python scripts/prof_solve.py kernels 2>&1 | grep -v "^=========     " | head -30
