#!/bin/bash
# Switch the blocked kernel to 12-qubit tiles, 256 threads, one CTA per SM (experiment).
sed -i 's/constexpr int kTileQubitsMax = 11;/constexpr int kTileQubitsMax = 12;/; s/constexpr int kThreadBits = 7;/constexpr int kThreadBits = 8;/' paper_2310_17739_b200/csrc/planner.h
sed -i 's/__launch_bounds__(kPassThreads, 2) k_blocked/__launch_bounds__(kPassThreads, 1) k_blocked/' paper_2310_17739_b200/csrc/device.cu
make -s -C paper_2310_17739_b200/csrc 2>&1 | grep -E "error" ; grep -A3 k_blocked paper_2310_17739_b200/csrc/build/device.ptxas.txt | sed -n 3,4p
