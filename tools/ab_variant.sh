# A/B of an in-tree build variant (libnucsim_b200_<v>.so) against the default
# usage: bash tools/ab_variant.sh <variant> [cfg...]
v=$1; shift
mkdir -p gpurun_out
for cfg in ${@:-deep21 rand28}; do
  for lib in default $v; do
    env $( [ $lib = default ] || echo NSB_LIB_VARIANT=$lib ) python bench.py --config $cfg --no-cpu-baseline --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/abv_${cfg}_$lib.log 2>&1
    echo "$cfg $lib $(tail -1 gpurun_out/abv_${cfg}_$lib.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["fp64"]["frac"], d["roofline"]["frac"])' 2>&1 | tail -1)"
  done
done
