cat > /tmp/pm.py <<'PY'
import os, sys
sys.argv = ["prof_mr.py", "--workload", "cfg3", "--warmup", "4", "--steps", "2"]
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import bench
from paper_1603_05211_b200 import mr as M
orig = M.MRSolver.build
def build(self, aos):
    self.set_numerics(True)
    return orig(self, aos)
M.MRSolver.build = build
exec(open("tools/prof_mr.py").read())
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3t_launches.csv python /tmp/pm.py > gpurun_out/c3t_l.log 2>&1; tail -1 gpurun_out/c3t_l.log
