#!/bin/bash
# Round-2 evidence for profiles/ (one B200): bench lines first, then ncu.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python bench.py --steps 5 --warmup 3 > gpurun_out/f_deep21.log 2>&1 || exit 1
for c in rand28 ucc8 mcm16; do
  python bench.py --config $c --steps 5 --warmup 3 --no-sharded > gpurun_out/f_$c.log 2>&1
done
python bench.py --trotter 913 --steps 1 --warmup 1 --no-cpu-baseline --no-sharded --e2e-steps 1 > gpurun_out/f_1e8.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sharded --e2e-steps 1 > gpurun_out/p_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_blocked -s 1 -c 1 \
    -o gpurun_out/p_full python bench.py --trotter 1 --steps 1 --warmup 1 --no-cpu-baseline \
    --no-sharded --e2e-steps 1 > gpurun_out/p_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_blocked -s 3 -c 1 \
    -o gpurun_out/p_full_rand28 python bench.py --config rand28 --steps 1 --warmup 3 --no-cpu-baseline \
    --no-sharded --e2e-steps 1 > gpurun_out/p_full_rand28.log 2>&1
for cfg in deep21 rand28; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_blocked \
      -s 3 -c 1 --csv --log-file gpurun_out/dram_$cfg.csv \
      python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline --no-sharded --e2e-steps 1 \
      > gpurun_out/dram_$cfg.log 2>&1
done
echo profile-done
