# Quick GPU iteration: the PCG / field / step parity tests, then the config-4
# bench (step only) with the cluster and the per-site mat-vec.
# usage: bash tools/gpu_quick.sh TAG [pytest -k expression]
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${1:-q}; K=${2:-"pcg or polar or field or tmatvec or amoeba or fullsize"}
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
timeout 400 python bench.py --no-cpu-baseline --no-md --no-recip --no-polar-forces > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo rc=$? >> gpurun_out/${T}_bench.err
MDG_CLUSTER_MATVEC=0 timeout 400 python bench.py --no-cpu-baseline --no-md --no-recip --no-polar-forces > gpurun_out/${T}_bench_site.json 2> gpurun_out/${T}_bench_site.err
tail -n 3 gpurun_out/${T}_tests.log
