"""Times the device AMR run against the reference's on the same host (args:
dim base level steps dt kind [integrator flux] [ref])."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1603_05211_b200 import amr
from paper_1603_05211_b200.uniform import SchemeConfig

dim, base, level, steps = (int(x) for x in sys.argv[1:5])
dt = float(sys.argv[5]); kind = int(sys.argv[6])
integ = int(sys.argv[7]) if len(sys.argv) > 7 else 1
flux = int(sys.argv[8]) if len(sys.argv) > 8 else 1
with_ref = len(sys.argv) > 9 and sys.argv[9] == "ref"
opts = amr.AmrOptions(max_levels=level - base)
h = amr.PatchHierarchy(dim, base, opts, scheme=SchemeConfig(flux, 1, integ))
t0 = time.time(); h.initialize_case(kind, 1); t_init = time.time() - t0
per = 1 << (level - base)
h.run(per, dt)  # warm-up cycle
u0 = h.cell_updates(); l0 = h.kernel_launches(); r0 = h.remesh_stats()
t0 = time.time(); rep = h.run(steps, dt); wall = time.time() - t0
upd = h.cell_updates() - u0
print(f"gpu: init {t_init:.3f}s run {wall:.3f}s steps {steps} updates {upd} -> {upd / wall:.4e} cell-updates/s "
      f"launches {h.kernel_launches() - l0} boxes {[h.level_info(l)[0] for l in range(h.n_levels())]} "
      f"cells {rep.cells_per_step[-1]} max_cfl {rep.max_cfl:.3f} remesh {h.remesh_stats()[0] - r0[0]:.3f}s "
      f"in {h.remesh_stats()[1] - r0[1]} calls")
if with_ref:
    from oracle import oracle
    r = oracle.ref_amr_run(dim, level, base, steps + per, dt, case_kind=kind, seed=1, flux=flux, integrator=integ)
    print(f"ref: wall {r['wall_seconds']:.3f}s for {steps + per} steps err {r['err_kind']} {r['err'][:60]}")
