"""B200-native drop-in for the gate-application path of arXiv 2310.17739's
reference simulator (``nucsim`` 0.1.0).

Same names and semantics as the reference's hot-path API
(nucsim/__init__.py:10-76 restricted to the circuit IR, gate vocabulary,
fusion, engine and the OpenQASM reader): a program written against ``nucsim``'s ``Circuit`` /
``fuse_pipeline`` / ``run`` runs unchanged with this package imported in its
place.  Fusion executes natively on the host (csrc/fusion.cpp); every state
operation executes on the GPU through libnucsim_b200.so (csrc/device.cu).
"""

from .circuit import Circuit, Instruction
from .errors import (DegenerateSpectrumError, FilterAssertionError, MmaStructureError,
                     NucsimError, ProjectionError, QasmError, ResourceLimitError,
                     SpectrumGuardError)
from .fusion import (FusionStats, PassStats, absorb_1q, fuse_2q, fuse_pipeline, gate_count,
                     merge_1q, normalize_2q_order)
from .gates import Gate, gate_matrix
from .pauli import PauliHamiltonian
from .qasm import parse_qasm, parse_qasm_packed
from .engine import (EPS_MMA, RunReport, StateVector, apply_1q, apply_2q, apply_dense,
                     assert_measure, bitstring, expectation_pauli, infer_ancilla,
                     measure_project, run, sample, success_product)

__version__ = "0.1.0"
