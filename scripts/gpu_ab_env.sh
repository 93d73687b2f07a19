# A/B of solve/setup time: the same lib with env setting $ENVB vs default
cd $GRAFT_REPO_ROOT
for spec in ${SPECS:-randk3d:160,160,160,0}; do
 for r in 1 2; do
  SPEC=$spec TAG=default REPS=${REPS:-8} timeout 600 python scripts/time_setup.py 2>&1 | tail -1
  env $ENVB SPEC=$spec TAG="$ENVB" REPS=${REPS:-8} timeout 600 python scripts/time_setup.py 2>&1 | tail -1
 done
done
