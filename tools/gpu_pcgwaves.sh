# PCG tests, then the config-4 step at several PCG mat-vec wave counts
# (MDG_PCG_WAVES; 0 = the default 16).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=$1
timeout 900 python -m pytest tests -m gpu -x -q -k "pcg or amoeba or fullsize or polar or dd or md" > gpurun_out/${T}_tests.log 2>&1; echo rc=$? >> gpurun_out/${T}_tests.log
tail -n 2 gpurun_out/${T}_tests.log
for w in 0 1 2 4; do
  MDG_PCG_WAVES=$w timeout 400 python bench.py --no-cpu-baseline --no-md --no-recip --no-polar-forces --no-e2e > gpurun_out/${T}_bench_w$w.json 2> gpurun_out/${T}_bench_w$w.err
  python -c "
import json;d=json.load(open('gpurun_out/${T}_bench_w$w.json'));r=d['roofline']
print('w$w', round(d['ms_per_step'],3), r['kernel'], r['avg_launch_ms'], r['frac'], {k:v['avg_launch_ms'] for k,v in d['roofline_other_kernels'].items()})" || tail -n 5 gpurun_out/${T}_bench_w$w.err
done
MDG_PROFILE_STEP=1 timeout 300 python tools/one_step.py 4 1 > gpurun_out/${T}_onestep.log 2>&1; tail -c 600 gpurun_out/${T}_onestep.log
