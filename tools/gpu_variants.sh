# Bench (step only) of kernel-variant libraries built as
# paper_1906_01211_b200/libmdg_<v>.so (make OBJ=... LIB=... EXTRA=-D...).
# usage: bash tools/gpu_variants.sh TAG "v1 v2 ..." [pytest -k expr for the default library]
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=$1; V=$2; K=$3
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
  tail -n 3 gpurun_out/${T}_tests.log
fi
for v in $V; do
  if [ "$v" = "default" ]; then L=""; else L=$PWD/paper_1906_01211_b200/libmdg_$v.so; fi
  env ${L:+MDG_LIB=$L} timeout 400 python bench.py --no-cpu-baseline --no-md --no-recip --no-polar-forces --no-e2e > gpurun_out/${T}_bench_$v.json 2> gpurun_out/${T}_bench_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/${T}_bench_$v.json'));r=d['roofline']
print('$v', round(d['ms_per_step'],3), r['kernel'], r['avg_launch_ms'], r['frac'], {k:v['avg_launch_ms'] for k,v in d['roofline_other_kernels'].items()})" || tail -n 5 gpurun_out/${T}_bench_$v.err
done
