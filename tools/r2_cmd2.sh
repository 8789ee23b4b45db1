bash tools/r2_overlap.sh 2
NO_TESTS=1 bash tools/r2_ab.sh "deep21 rand28" base
