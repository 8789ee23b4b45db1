"""Full-size (BASELINE config 3, 21 qubits) properties of the device path,
where the oracle is too slow to compare amplitude by amplitude:

* the fused gate stream of the P9-shaped filter circuit followed by its
  adjoint (reversed, conjugate-transposed payloads) returns |0...0>;
* the single-launch MMA program and the host-driven item path (per-op
  measurement kernels) agree on every assertion probability;
* edge cases: empty programs, one-qubit states, marker-only circuits."""

import numpy as np
import pytest

from paper_2310_17739_b200 import _native as N
from paper_2310_17739_b200 import workloads as W
from paper_2310_17739_b200.engine import DeviceProgram, StateVector, _branch_probability, _project
from paper_2310_17739_b200.gates import BY_CODE, Gate, gate_matrix

pytestmark = pytest.mark.gpu


def _matrix(rec, params, pool):
    nq = int(rec["nq"])
    if int(rec["payload"]) >= 0:
        d = 1 << nq
        off = int(rec["payload"])
        return pool[off: off + d * d].reshape(d, d)
    g = BY_CODE[int(rec["tag"])]
    p0 = int(rec["param"])
    return gate_matrix(g, tuple(params[p0: p0 + g.n_params]) if g.n_params else ())


def _adjoint(ops, params, pool):
    """Reversed stream of payload gates U^dagger (C1 / C2 tags)."""
    gates = ops[ops["kind"] == N.OP_GATE][::-1]
    out = np.zeros(len(gates), N.OP_DTYPE)
    mats = []
    off = 0
    for i, rec in enumerate(gates):
        u = np.conj(_matrix(rec, params, pool)).T
        nq = int(rec["nq"])
        out[i]["kind"], out[i]["nq"], out[i]["cbit"] = N.OP_GATE, nq, -1
        out[i]["tag"] = (Gate.C1 if nq == 1 else Gate.C2).code
        out[i]["q"] = rec["q"]
        out[i]["mask"] = rec["mask"]
        out[i]["src"], out[i]["param"], out[i]["payload"] = -1, -1, off
        mats.append(np.ascontiguousarray(u).reshape(-1))
        off += u.size
    return out, np.concatenate(mats)


def test_filter21_stream_then_adjoint_is_identity():
    wl = W.filter_workload(20, trotter=1, n_steps=2, n_scatter=8, trial="10" * 10)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    gates = fops[fops["kind"] == N.OP_GATE]
    inv, inv_pool = _adjoint(gates, wl.params, pool)
    state = StateVector(wl.n_qubits)
    fwd = DeviceProgram(state, gates, wl.params, pool)
    assert fwd.info.n_passes > 100
    fwd.run_mma()
    mid = state.amps.copy()
    assert abs(np.linalg.norm(mid) - 1.0) < 1e-10
    assert abs(mid[0]) < 0.99  # the stream moved the state
    back = DeviceProgram(state, inv, np.zeros(1), inv_pool)
    back.run_mma()
    a = state.amps
    assert abs(a[0] - 1.0) < 1e-9
    assert np.linalg.norm(a[1:]) < 1e-9


def test_filter21_mma_launch_matches_item_path():
    wl = W.filter_workload(20, trotter=1, n_steps=8, n_scatter=8, trial="10" * 10)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    state = StateVector(wl.n_qubits)
    prog = DeviceProgram(state, exe, wl.params, pool)
    p_mma = prog.run_mma()
    final_mma = state.amps.copy()
    state.restart()
    p_items = []
    for i, (kind, q, step) in enumerate(prog.items()):
        if kind == N.OP_MEASURE:
            p0 = _branch_probability(state, q, 0)
            p_items.append(p0 * prog.p0_scale(step))
            _project(state, q, 0, p0)
        elif kind == N.OP_GATE:
            prog.run_item(i)
    assert len(p_mma) == 8
    np.testing.assert_allclose(p_mma, p_items, rtol=1e-12, atol=0)
    a = state.amps
    assert np.linalg.norm(a - final_mma) <= 1e-10 * np.linalg.norm(a)


def test_empty_and_marker_only_programs():
    state = StateVector(8)
    empty = np.zeros(0, N.OP_DTYPE)
    prog = DeviceProgram(state, empty, np.zeros(1), np.zeros(1, np.complex128))
    assert prog.run_mma() == []
    assert state.amps[0] == 1.0
    ops = np.zeros(2, N.OP_DTYPE)
    ops["kind"] = (N.OP_MEASURE, N.OP_RESET)
    ops["nq"], ops["cbit"], ops["src"], ops["param"], ops["payload"] = 1, -1, -1, -1, -1
    ops["q"] = -1
    ops["q"][:, 0] = 3
    prog = DeviceProgram(state, ops, np.zeros(1), np.zeros(1, np.complex128))
    assert prog.run_mma() == [1.0]


@pytest.mark.parametrize("n", [1, 2, 5])
def test_tiny_states_through_the_plan(n):
    """n < 6 takes the per-op path of the same plan API."""
    rng = np.random.default_rng(n)
    ops = np.zeros(6, N.OP_DTYPE)
    params = []
    for i in range(6):
        ops[i]["kind"], ops[i]["tag"], ops[i]["nq"], ops[i]["cbit"] = N.OP_GATE, Gate.U3.code, 1, -1
        ops[i]["q"] = (i % n, -1, -1, -1, -1)
        ops[i]["src"], ops[i]["payload"], ops[i]["param"] = -1, -1, len(params)
        params.extend(rng.uniform(-3, 3, 3))
    params = np.asarray(params)
    state = StateVector(n)
    DeviceProgram(state, ops, params, np.zeros(1, np.complex128)).run_mma()
    want = np.zeros(1 << n, complex)
    want[0] = 1
    for rec in ops:
        u = gate_matrix(Gate.U3, tuple(params[int(rec["param"]): int(rec["param"]) + 3]))
        q = int(rec["q"][0])
        want = want.reshape(-1, 2, 1 << q)
        want = np.einsum("ab,rbt->rat", u, want).reshape(-1)
    np.testing.assert_allclose(state.amps, want, atol=1e-13)


@pytest.mark.parametrize("n", [25])
def test_hbm_regime_layered_stream_then_adjoint_is_identity(n):
    """Above the L2-resident size (tiles hold qubits 0..2, 128-byte runs) the
    random layered circuit of BASELINE config 4 followed by its adjoint
    returns |0...0>; 512 MiB state, every pass streams HBM."""
    wl = W.layered_workload(n, 6, 2310)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    gates = fops[fops["kind"] == N.OP_GATE]
    inv, inv_pool = _adjoint(gates, wl.params, pool)
    state = StateVector(n)
    fwd = DeviceProgram(state, gates, wl.params, pool)
    fwd.run_mma()
    assert abs(state.norm() - 1.0) < 1e-10
    back = DeviceProgram(state, inv, np.zeros(1), inv_pool)
    back.run_mma()
    a = state.amps
    assert abs(a[0] - 1.0) < 1e-10
    assert np.linalg.norm(a[1:]) < 1e-10


def test_state_released_before_its_programs():
    """Python may collect a StateVector (its nsb_ctx) before the DeviceProgram
    built on it: the plan holds a reference on the context, so destroying the
    plan afterwards is safe (regression: segfault in nsb_plan_destroy during
    garbage collection, round 1)."""
    import gc
    wl = W.filter_workload(11, trotter=1, n_steps=2, trial="10" * 5 + "1")
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    state = StateVector(12)
    progs = [DeviceProgram(state, exe, wl.params, pool) for _ in range(3)]
    progs[0].run_mma()
    state._dev.close()  # the owner's reference goes first
    del state
    gc.collect()
    for p in progs:
        p.__del__()
    gc.collect()


def test_plan_rejects_a_resized_state():
    """A plan is bound to the qubit count it was built for (no out-of-bounds
    run after nsb_state_init changes the state size)."""
    wl = W.layered_workload(12, 2, 3)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    state = StateVector(12)
    prog = DeviceProgram(state, fops, wl.params, pool)
    state._dev.call("nsb_state_init", 10)
    with pytest.raises(ValueError):
        prog.run_mma()


def test_null_status_still_reports_assertion_failure():
    """nsb_plan_run_mma returns NSB_EASSERT when the caller passes no status."""
    import ctypes
    c = np.zeros(4, N.OP_DTYPE)
    c["cbit"], c["src"], c["param"], c["payload"] = -1, -1, -1, -1
    c["q"] = -1
    c[0]["kind"], c[0]["tag"], c[0]["nq"], c[0]["q"][0] = N.OP_GATE, Gate.X.code, 1, 3
    c[1]["kind"], c[1]["nq"], c[1]["q"][0] = N.OP_MEASURE, 1, 3
    c[2]["kind"], c[2]["nq"], c[2]["q"][0] = N.OP_RESET, 1, 3
    c[3]["kind"], c[3]["tag"], c[3]["nq"], c[3]["q"][0] = N.OP_GATE, Gate.H.code, 1, 0
    state = StateVector(8)
    prog = DeviceProgram(state, c, np.zeros(1), np.zeros(1, np.complex128))
    probs = np.zeros(1)
    code = N.lib().nsb_plan_run_mma(state._dev.handle, prog.handle, ctypes.c_double(1e-12),
                                    N.ptr(probs), None)
    assert code == 2  # NSB_EASSERT


def test_streamed_mma_run_matches_the_single_launch_program():
    """nsb_run_mma_streamed (planning of part s+1 behind the device run of part
    s, one launch per part, p0 carried through the record) reproduces the
    single-launch MMA program: every p0 and the final state."""
    from paper_2310_17739_b200.engine import run_mma_streamed
    wl = W.filter_workload(20, trotter=1, n_steps=8, n_scatter=8, trial="10" * 10)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    state = StateVector(wl.n_qubits)
    prog = DeviceProgram(state, exe, wl.params, pool)
    p_one = prog.run_mma()
    a_one = state.amps.copy()
    state.restart()
    p_str = run_mma_streamed(state, exe, wl.params, pool)
    assert len(p_str) == 8
    # the streamed run cuts the first gate run into shorter parts (exact frame
    # flushes), so group boundaries -- and roundings -- differ slightly
    np.testing.assert_allclose(p_str, p_one, rtol=0, atol=1e-12)
    assert np.linalg.norm(state.amps - a_one) <= 1e-11
    assert state.last_device_ms > 0.0


def test_streamed_mma_assertion_failure():
    """A failed assertion in a streamed run stops the later launches and raises
    FilterAssertionError(step, p0) like the single-launch program."""
    from paper_2310_17739_b200.engine import run_mma_streamed
    from paper_2310_17739_b200.errors import FilterAssertionError
    rng = np.random.default_rng(3)
    n = 8
    ops = []
    params = []

    def gate(tag, qs, ps=()):
        rec = np.zeros(1, N.OP_DTYPE)[0]
        rec["kind"], rec["tag"], rec["nq"], rec["cbit"] = N.OP_GATE, tag.code, len(qs), -1
        rec["q"] = tuple(qs) + (-1,) * (5 - len(qs))
        rec["src"], rec["payload"] = -1, -1
        rec["param"] = len(params) if ps else -1
        params.extend(ps)
        ops.append(rec)

    def marker(kind, q):
        rec = np.zeros(1, N.OP_DTYPE)[0]
        rec["kind"], rec["nq"], rec["cbit"] = kind, 1, -1
        rec["q"] = (q, -1, -1, -1, -1)
        rec["src"], rec["param"], rec["payload"] = -1, -1, -1
        ops.append(rec)

    for step in range(3):
        for _ in range(20):
            a, b = (int(x) for x in rng.choice(n - 1, 2, replace=False))
            gate(Gate.RZZ, (a, b), (float(rng.uniform(-1, 1)),))
            gate(Gate.U3, (a,), tuple(float(x) for x in rng.uniform(-1, 1, 3)))
        if step == 1:
            gate(Gate.X, (n - 1,))  # the ancilla is |1>: P(|0>) = 0 at step 1
        marker(N.OP_MEASURE, n - 1)
        marker(N.OP_RESET, n - 1)
    ops = np.array(ops, N.OP_DTYPE)
    state = StateVector(n)
    with pytest.raises(FilterAssertionError) as e:
        run_mma_streamed(state, ops, np.asarray(params or [0.0]), np.zeros(1, np.complex128))
    assert e.value.step == 1


@pytest.mark.parametrize("shape", ["leading_markers", "gates_only", "back_to_back"])
def test_streamed_mma_edge_shapes(shape):
    """Parts without gates (markers first, consecutive assertions) and circuits
    without markers run the same through the streamed call as through the
    single-launch program."""
    from paper_2310_17739_b200.engine import run_mma_streamed
    rng = np.random.default_rng(11)
    n = 9
    recs, params = [], []

    def gate(qs):
        rec = np.zeros(1, N.OP_DTYPE)[0]
        rec["kind"], rec["tag"], rec["nq"], rec["cbit"] = N.OP_GATE, Gate.U3.code, 1, -1
        if len(qs) == 2:
            rec["tag"], rec["nq"] = Gate.CU3.code, 2
        rec["q"] = tuple(qs) + (-1,) * (5 - len(qs))
        rec["src"], rec["payload"], rec["param"] = -1, -1, len(params)
        params.extend(rng.uniform(-0.4, 0.4, 3))
        recs.append(rec)

    def marker(kind):
        rec = np.zeros(1, N.OP_DTYPE)[0]
        rec["kind"], rec["nq"], rec["cbit"] = kind, 1, -1
        rec["q"] = (n - 1, -1, -1, -1, -1)
        rec["src"], rec["param"], rec["payload"] = -1, -1, -1
        recs.append(rec)

    def block(count):
        for _ in range(count):
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            gate((a, b) if rng.random() < 0.6 else (a,))

    if shape == "leading_markers":
        marker(N.OP_MEASURE)
        marker(N.OP_RESET)
        block(60)
        marker(N.OP_MEASURE)
        marker(N.OP_RESET)
    elif shape == "gates_only":
        block(120)
    else:
        block(40)
        marker(N.OP_MEASURE)
        marker(N.OP_RESET)
        marker(N.OP_MEASURE)
        marker(N.OP_RESET)
        block(40)
    ops = np.array(recs, N.OP_DTYPE)
    params = np.asarray(params)
    state = StateVector(n)
    want_p = DeviceProgram(state, ops, params, np.zeros(1, np.complex128)).run_mma()
    want = state.amps.copy()
    state.restart()
    got_p = run_mma_streamed(state, ops, params, np.zeros(1, np.complex128))
    np.testing.assert_allclose(got_p, want_p, rtol=0, atol=1e-14)
    assert np.linalg.norm(state.amps - want) <= 1e-12
