# A/B of planner/kernel env settings on one config: bash tools/ab_env.sh cfg "ENV=1" ["ENV2=1 ENV3=0" ...]
cfg=$1; shift
mkdir -p gpurun_out
for v in default "$@"; do
  tag=$(echo "$v" | tr ' =' '__')
  env $( [ "$v" = default ] || echo $v ) python bench.py --config $cfg --no-cpu-baseline --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/abe_${cfg}_$tag.log 2>&1
  echo "$cfg [$v] $(tail -1 gpurun_out/abe_${cfg}_$tag.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], "passes", d["config"]["passes"], "frac", d["roofline"]["frac"])' 2>&1 | tail -1)"
done
