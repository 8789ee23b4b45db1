#!/bin/bash
# Profiling evidence for profiles/ (run under gpurun on one B200).
#  1. plain bench (must exit 0 before any ncu run)
#  2. ncu launch list of the same command (per-launch device time, cold cache)
#  3. ncu --set full of k_blocked on the 1-Trotter-slice variant of the workload
set -e
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_launch.log 2>&1
python bench.py --trotter 1 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof_small.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_blocked -s 1 -c 1 \
    -o gpurun_out/prof_full python bench.py --trotter 1 --steps 1 --warmup 1 --no-cpu-baseline \
    --e2e-steps 1 > gpurun_out/prof_full.log 2>&1

# 4. DRAM bytes of one full-workload k_blocked launch per config (roofline "traffic")
for cfg in deep21 rand28; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_blocked \
      -s 3 -c 1 --csv --log-file gpurun_out/dram_$cfg.csv \
      python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      > gpurun_out/dram_$cfg.log 2>&1
done
echo dram-done
echo profile-done
