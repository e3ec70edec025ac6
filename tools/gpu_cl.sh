# Cluster-PCG iteration: parity tests, then the config-4 step with the
# cluster mat-vec for each library variant, and the per-site default.
# usage: bash tools/gpu_cl.sh TAG "v1 v2 ..."
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=$1; V=$2
MDG_CLUSTER_MATVEC=1 timeout 900 python -m pytest tests -m gpu -x -q -k "cluster or pcg or amoeba or fullsize" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
tail -n 2 gpurun_out/${T}_tests.log
for v in $V; do
  if [ "$v" = "default" ]; then L=""; else L=$PWD/paper_1906_01211_b200/libmdg_$v.so; fi
  env ${L:+MDG_LIB=$L} MDG_CLUSTER_MATVEC=1 timeout 400 python bench.py --no-cpu-baseline --no-md --no-recip --no-polar-forces --no-e2e > gpurun_out/${T}_bench_$v.json 2> gpurun_out/${T}_bench_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/${T}_bench_$v.json'));r=d['roofline']
print('$v', round(d['ms_per_step'],3), r['kernel'], r['avg_launch_ms'], r['frac'], {k:v['avg_launch_ms'] for k,v in d['roofline_other_kernels'].items()})" || tail -n 5 gpurun_out/${T}_bench_$v.err
done
