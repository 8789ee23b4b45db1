# A/B of payload classification: default (near-zero cleaning + real Pair classes),
# real classes off, exact-zero rule only.  usage: bash tools/ab_classes.sh [cfg...]
mkdir -p gpurun_out
for cfg in ${@:-deep21 rand28}; do
  for v in default NSB_NO_GROUP_FUSION=1 NSB_NO_REAL_CLASSES=1; do
    env $( [ $v = default ] || echo $v ) python bench.py --config $cfg --no-cpu-baseline --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/ab_${cfg}_${v%%=*}.log 2>&1
    echo "$cfg $v $(tail -1 gpurun_out/ab_${cfg}_${v%%=*}.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["fp64"]["frac"])' 2>&1 | tail -1)"
  done
done
