#!/bin/bash
# The reference's own test suite against this package on a B200 (see
# tools/reference_suite.py; run `python tools/reference_suite.py prepare` in the
# build container first -- baseline/ travels with the gpurun snapshot).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
cd baseline/_refpkg/tests || exit 1
timeout 2400 python -m pytest -q -rfE -p no:cacheprovider --durations=15 \
  test_engine.py test_fusion.py test_acceptance.py test_gates.py test_circuit.py test_cli.py \
  test_qasm.py test_projection.py test_hamiltonian.py test_lcu.py \
  > ../../../gpurun_out/refsuite.log 2>&1
echo "refsuite rc=$?" >> ../../../gpurun_out/refsuite.log
tail -40 ../../../gpurun_out/refsuite.log
