"""Kernel times of the config-4 AMOEBA step with reciprocal-space Ewald
(smooth PME 216^3, order 5, the bench's with_ewald_recip line), profile mode."""
import sys
sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.Workload(4, 0, 1)
wl.eng.set_ewald_recip((216, 216, 216), 5)
for _ in range(3):
    wl.step()
wl.eng.profile(True)
wl.step()
wl.step()
wl.eng.synchronize()
rep = wl.eng.profile_report()
tot = sum(v[1] for v in rep.values())
for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1])[:30]:
    print(k, v[0], round(v[1], 3))
print("total (2 steps)", round(tot, 3))
