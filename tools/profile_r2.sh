#!/bin/bash
# Round-2 profiling evidence (one B200): plain runs first, then ncu.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/p_plain.log 2>&1 || exit 1
for c in ucc8 mcm16; do
  for v in 0 1; do
    env $( [ $v = 1 ] && echo NSB_FULL_GRID=1 ) python bench.py --config $c --steps 5 --warmup 3 \
       --no-cpu-baseline --e2e-steps 1 > gpurun_out/p_${c}_fullgrid$v.log 2>&1
  done
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/p_launch.log 2>&1
python bench.py --trotter 1 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/p_small.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_blocked -s 1 -c 1 \
    -o gpurun_out/p_full python bench.py --trotter 1 --steps 1 --warmup 1 --no-cpu-baseline \
    --e2e-steps 1 > gpurun_out/p_full.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum --clock-control none -k regex:k_blocked \
    -s 3 -c 1 --csv --log-file gpurun_out/dram_deep21.csv \
    python bench.py --config deep21 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/dram_deep21.log 2>&1
echo profile-done
