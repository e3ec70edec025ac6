# Run the step bench under several env / flag variants; print rc + last error.
# usage: bash tools/gpu_bisect.sh TAG "name|ENV=V,ENV2=V|--flag --flag2" ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=$1; shift
for spec in "$@"; do
  IFS='|' read -r name envs flags <<< "$spec"
  E=$(echo "$envs" | tr ',' ' ')
  env $E timeout 240 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 $flags \
    > gpurun_out/${T}_$name.json 2> gpurun_out/${T}_$name.err
  echo "$name rc=$? $(grep -h 'Error' gpurun_out/${T}_$name.err | tail -n 1 | cut -c1-160)"
done
