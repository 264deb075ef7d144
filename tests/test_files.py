"""Files on the path, CPU only: Matrix Market IO,
the excitation-JSON "files" problem class, and the shortest round-trip CSV
writers.  Each test restates one of the reference's own tests
(proj/tests/test_matrix_market.cpp, proj/tests/test_config_io.cpp)."""
import csv

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1905_13076_b200 as ps


def _write(path, text):
    path.write_text(text)
    return str(path)


def test_write_read_round_trip_is_bitwise(tmp_path):
    """test_matrix_market.cpp:39-58."""
    rng = np.random.default_rng(123)
    for _ in range(5):
        dense = rng.uniform(-1, 1, size=(6, 4))
        dense[0, 0] = 0.0
        dense[3, 2] = 1e-17
        dense[5, 3] = -3.0e8
        m = sp.csr_matrix(dense)
        m.eliminate_zeros()
        path = str(tmp_path / "roundtrip.mtx")
        ps.write_matrix_market(path, m)
        back = ps.read_matrix_market(path)
        assert back.shape == m.shape
        assert np.array_equal(back.toarray(), m.toarray())


def test_symmetric_storage_expands(tmp_path):
    """test_matrix_market.cpp:60-78."""
    path = _write(tmp_path / "sym.mtx", "%%MatrixMarket matrix coordinate real symmetric\n% lower triangle only\n"
                                        "3 3 4\n1 1 2.5\n2 1 -1.0\n3 2 0.25\n3 3 4.0\n")
    d = ps.read_matrix_market(path).toarray()
    assert d[0, 0] == 2.5 and d[0, 1] == -1.0 and d[1, 0] == -1.0 and d[1, 2] == 0.25 and d[1, 1] == 0.0
    assert np.array_equal(d, d.T)


def test_duplicates_summed_and_header_case(tmp_path):
    """test_matrix_market.cpp:80-104."""
    path = _write(tmp_path / "dup.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n1 1 2.0\n"
                                        "2 2 -1.0\n")
    m = ps.read_matrix_market(path)
    assert m[0, 0] == 3.0 and m[1, 1] == -1.0
    path = _write(tmp_path / "case.mtx", "%%MatrixMarket MATRIX Coordinate REAL General\n% comment\n"
                                         "%another comment\n1 1 1\n1 1 7.0\n")
    assert ps.read_matrix_market(path)[0, 0] == 7.0


@pytest.mark.parametrize("text", [
    "%%NotMatrixMarket matrix coordinate real general\n1 1 1\n1 1 1.0\n",
    "%%MatrixMarket matrix array real general\n2 2\n1.0\n0.0\n0.0\n1.0\n",
    "%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 x 1.0\n",
])
def test_malformed_input_rejected(tmp_path, text):
    """test_matrix_market.cpp:106-140."""
    with pytest.raises(ps.ParasteadyError, match="matrix_market"):
        ps.read_matrix_market(_write(tmp_path / "bad.mtx", text))
    with pytest.raises(ps.ParasteadyError, match="cannot open"):
        ps.read_matrix_market(str(tmp_path / "nope.mtx"))


def _dae_files(tmp_path):
    ref = ps.build_dae_pair()
    ps.write_matrix_market(str(tmp_path / "mass.mtx"), ref.csr(ref.mass_values))
    ps.write_matrix_market(str(tmp_path / "stiffness.mtx"), ref.csr(ref.stiffness_values))
    _write(tmp_path / "excitation.json", '{"period": 0.02,\n "terms": [{"amplitude": 1.0, "frequency": 50.0,\n'
                                         '            "dofs": [0], "values": [1.0]}]}')
    return ref, [str(tmp_path / f) for f in ("mass.mtx", "stiffness.mtx", "excitation.json")]


def test_load_problem_reproduces_the_dae_pair(tmp_path):
    """test_matrix_market.cpp:142-167 (matrices bitwise, excitation bitwise)."""
    ref, files = _dae_files(tmp_path)
    loaded = ps.load_problem(*files)
    assert loaded.dim == 2 and loaded.is_linear()
    assert np.array_equal(loaded.csr(loaded.mass_values).toarray(), ref.csr(ref.mass_values).toarray())
    assert np.array_equal(loaded.csr(loaded.stiffness_values).toarray(), ref.csr(ref.stiffness_values).toarray())
    assert loaded.period == ref.period
    t_ref, t_new = ref.excitation_terms(), loaded.excitation_terms()
    assert len(t_ref) == len(t_new) == 1
    for a, b in zip(t_ref, t_new):
        assert np.array_equal(a["pattern"], b["pattern"])
        assert a["amplitude"] == b["amplitude"] and a["frequency"] == b["frequency"] and a["phase"] == b["phase"]


def test_load_problem_rejects_inconsistent_inputs(tmp_path):
    """test_matrix_market.cpp:169-194 and parse_excitation_text's messages."""
    ref, (m, k, f) = _dae_files(tmp_path)
    ps.write_matrix_market(str(tmp_path / "k3.mtx"), sp.identity(3, format="csr"))
    with pytest.raises(ps.ParasteadyError, match="do not match"):
        ps.load_problem(m, str(tmp_path / "k3.mtx"), f)
    asym = _write(tmp_path / "asym.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n1 2 0.5\n"
                                         "2 2 1.0\n")
    with pytest.raises(ps.ParasteadyError, match="not symmetric"):
        ps.load_problem(asym, k, f)
    with pytest.raises(ps.ParasteadyError, match="cannot open excitation file"):
        ps.load_problem(m, k, str(tmp_path / "nope.json"))
    for text, msg in (('{"period": 0.02, "terms": [], "x": 1}', "unknown excitation key"),
                      ('{"terms": []}', "numeric \"period\""),
                      ('{"period": 0.02, "terms": [{"amplitude": 1, "frequency": 50, "dofs": [5], "values": [1]}]}',
                       "out of range"),
                      ('{"period": 0.02, "terms": [{"amplitude": 1, "frequency": 75, "dofs": [0], "values": [1]}]}',
                       "integer multiple"),
                      ('{"period": 0.02, "terms": [{"amplitude": 1, "frequency": 50, "dofs": [0]}]}',
                       "matching dofs/values"),
                      ('{"period": 0.02, "terms": [', "parse error")):
        bad = _write(tmp_path / "bad.json", text)
        with pytest.raises(ps.ParasteadyError, match=msg):
            ps.load_problem(m, k, bad)


def test_format_double_round_trips_bitwise():
    """test_config_io.cpp:265-277."""
    rng = np.random.default_rng(71)
    xs = np.ldexp(rng.uniform(-1, 1, 200), rng.integers(-300, 301, 200))
    for x in list(xs) + [0.0, 1.0, -1.0, 0.1, 1e-17, -3.0e8, 0.02 / 3.0]:
        assert float(ps.format_double(x)) == x


def test_trajectory_and_history_files(tmp_path):
    """test_config_io.cpp:279-306."""
    mesh = ps.TimeMesh(4, 2, 0.02)
    states = np.array([[0.1 * n, -1.0 / (n + 1)] for n in range(4)])
    ps.write_trajectory_csv(str(tmp_path / "trajectory.csv"), states, mesh)
    rows = list(csv.reader(open(tmp_path / "trajectory.csv")))
    assert len(rows) == 5 and rows[0] == ["n", "t", "u0", "u1"]
    for n in range(4):
        row = rows[n + 1]
        assert int(row[0]) == n and float(row[1]) == mesh.boundary(n)
        assert float(row[2]) == states[n, 0] and float(row[3]) == states[n, 1]
    ps.write_history_csv(str(tmp_path / "history.csv"), [0.25, 1e-9], [0.5, 0.25])
    h = list(csv.reader(open(tmp_path / "history.csv")))
    assert len(h) == 3 and h[0] == ["k", "jump_norm", "wall_time_s"] and float(h[2][1]) == 1e-9
