# Timing decomposition of k_blocked (NSB_DEBUG_BLOCKED: 1 skip sweeps, 2 skip HBM, 3 both)
mkdir -p gpurun_out
for cfg in ${CFGS:-deep21 rand28}; do for d in ${DBGS:-0 1 2 3}; do
NSB_DEBUG_BLOCKED=$d python bench.py --config $cfg --no-cpu-baseline --e2e-steps 1 --steps 2 --warmup 3 > gpurun_out/dbg_${cfg}_$d.log 2>&1
echo "$cfg dbg=$d $(tail -1 gpurun_out/dbg_${cfg}_$d.log | cut -c1-300)"
done; done
