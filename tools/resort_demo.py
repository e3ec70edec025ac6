"""Locality lost and restored: config-4 step time (a) as uploaded (Morton
order), (b) after every molecule moved to another molecule's place (same
physical configuration, the stored order no longer follows space), (c) after
mdg_resort."""
import sys, os, json
sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '.'))
import numpy as np
import bench
wl = bench.Workload(4, 0, 1)
eng = wl.eng
def timed(k=10):
    wl.rebuild()
    for _ in range(2):
        wl.step()
    eng.synchronize()
    eng.timer_start()
    for _ in range(k):
        wl.step()
    ms = eng.timer_stop() / k
    e = eng.fetch_energies()[0]
    return ms, [float(x) for x in e[:3]]
out = {"as_uploaded": timed()}
n_mol = wl.n // 3
perm = np.random.default_rng(5).permutation(n_mol)
s = wl.sys
xyz = np.stack([s.x, s.y, s.z], 1).reshape(n_mol, 3, 3)[perm].reshape(-1, 3)
eng.upload_positions(xyz[:, 0], xyz[:, 1], xyz[:, 2])
out["scrambled_order"] = timed()
eng.synchronize()
eng.timer_start()
eng.resort()
out["resort_ms"] = eng.timer_stop()
out["after_resort"] = timed()
print(json.dumps(out))
