# Step bench under several environment settings / libraries.
# usage: bash tools/gpu_envs.sh TAG "name1:ENV=V,ENV2=V:lib name2::..." [pytest -k expr]
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=$1; V=$2; K=$3
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
  tail -n 2 gpurun_out/${T}_tests.log
fi
for spec in $V; do
  name=${spec%%:*}; rest=${spec#*:}; envs=${rest%%:*}; lib=${rest#*:}
  E=$(echo "$envs" | tr ',' ' ')
  if [ -n "$lib" ]; then E="$E MDG_LIB=$PWD/paper_1906_01211_b200/libmdg_$lib.so"; fi
  env $E timeout 400 python bench.py --no-cpu-baseline --no-md --no-recip --no-polar-forces --no-e2e > gpurun_out/${T}_bench_$name.json 2> gpurun_out/${T}_bench_$name.err
  python -c "
import json;d=json.load(open('gpurun_out/${T}_bench_$name.json'));r=d['roofline']
print('$name', round(d['ms_per_step'],3), r['avg_launch_ms'], {k:v['avg_launch_ms'] for k,v in d['roofline_other_kernels'].items()})" || tail -n 5 gpurun_out/${T}_bench_$name.err
done
