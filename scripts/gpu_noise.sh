cd $GRAFT_REPO_ROOT
st() { awk '/^cpu /{print "user",$2,"sys",$4,"idle",$5,"iowait",$6,"steal",$9}' /proc/stat; }
st; nproc; cat /proc/loadavg
timeout 900 python -m pytest tests -q -m gpu --durations=8 2>&1 | tail -12
st; cat /proc/loadavg
for i in 1 2 3; do REPS=8 python scripts/time_setup.py; done
st
ps aux --sort=-%cpu | head -8
