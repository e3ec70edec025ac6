"""Experiment: where the end-to-end step's extra milliseconds go (config 4):
device-resident steps vs + H2D upload vs + force fetch vs + energies fetch."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402

wl = bench.Workload(4, 0, 0)
eng = wl.eng
m = wl.m
xyz = m.host_array((3, wl.n))
xyz[0], xyz[1], xyz[2] = wl.sys.x, wl.sys.y, wl.sys.z
fbuf = m.host_array((3, wl.n))
eng.set_force_output(fbuf)
K = 10


def run(upload, fetch_f, fetch_e):
    for _ in range(2):
        eng.upload_positions(xyz[0], xyz[1], xyz[2])
        wl.step()
        eng.fetch_forces(out=fbuf)
    wl.rebuild()
    eng.synchronize()
    t0 = time.perf_counter()
    eng.timer_start()
    for k in range(K):
        if upload:
            eng.upload_positions(xyz[0], xyz[1], xyz[2])
        wl.step()
        if fetch_f:
            eng.fetch_forces(out=fbuf)
        if fetch_e:
            eng.fetch_energies()
    ms = eng.timer_stop()
    wall = (time.perf_counter() - t0) * 1e3
    return ms / K, wall / K


for args in [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, 1, 1), (0, 0, 0)]:
    print(args, [round(v, 3) for v in run(*args)], flush=True)
t0 = time.perf_counter()
for k in range(20):
    eng.upload_positions(xyz[0], xyz[1], xyz[2])
eng.synchronize()
print("upload only", round((time.perf_counter() - t0) * 1e3 / 20, 3), "ms", flush=True)
