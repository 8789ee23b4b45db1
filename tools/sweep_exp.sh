# Sweep decomposition: build variants first
#   make -C paper_2310_17739_b200/csrc OUT=../libnucsim_b200_noops.so BUILD=build_noops DEFS=-DNSB_SWEEP_NOOPS
#   make -C paper_2310_17739_b200/csrc OUT=../libnucsim_b200_nomem.so BUILD=build_nomem DEFS=-DNSB_SWEEP_NOMEM
# then: bash tools/sweep_exp.sh   (dbg=2: no global traffic)
mkdir -p gpurun_out
for cfg in deep21 rand28; do for v in default noops nomem; do
  for d in 0 2; do
    env NSB_DEBUG_BLOCKED=$d $( [ $v = default ] || echo NSB_LIB_VARIANT=$v ) python bench.py --config $cfg --no-cpu-baseline --e2e-steps 1 --steps 2 --warmup 2 > gpurun_out/sw_${cfg}_${v}_$d.log 2>&1
    echo "$cfg $v dbg=$d $(tail -1 gpurun_out/sw_${cfg}_${v}_$d.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])' 2>&1 | tail -1)"
  done
done; done
