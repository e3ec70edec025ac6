"""One AMOEBA step of a BASELINE config with the host-driven PCG loop
(profile mode), for ncu captures: python tools/one_step.py [config] [steps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = bench.Workload(cfg, 0, 1)
wl.eng.profile(True)
for _ in range(steps):
    wl.step()
wl.eng.synchronize()
print({k: (v[0], round(v[1], 3)) for k, v in wl.eng.profile_report().items()})
