"""CPU-only checks: the C-ABI library loads and exports every symbol the header declares, and
the host-side domain types / guards behave like the reference's (core.py, histogram.py)."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2005_03246_b200 as fcb
from paper_2005_03246_b200 import _lib

ROOT = Path(__file__).resolve().parent.parent


def header_functions():
    txt = (ROOT / "include" / "fastcdf_b200.h").read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fcg_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    names = header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.EXPORTED, f"{name} has no ctypes signature"
    assert lib.fcg_abi_version() == 1


def test_workspace_query_needs_no_gpu():
    """Size queries are pure host arithmetic (no device touched)."""
    import ctypes as C

    lib = _lib.load_library()
    nbytes = C.c_size_t(0)
    rc = lib.fcg_ecdf_grid(None, 1000, 3, None, None, _lib.i64_array([512, 512, 512]),
                           _lib.i32_array([1, 1, 1]), 0, 1, 0, None, None, C.byref(nbytes), None)
    assert rc == 0
    assert nbytes.value >= 512 ** 3 * 4  # int32 lattice of the exact output extents
    rc = lib.fcg_ecdf_grid(None, 10, 9, None, None, _lib.i64_array([2] * 9),
                           _lib.i32_array([1] * 9), 0, 1, 0, None, None, C.byref(nbytes), None)
    assert rc == _lib.FCG_EUNSUPPORTED
    assert b"dimension" in lib.fcg_last_error()


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    s = fcb.validate_sample([[0.1, 0.2], [0.3, 0.4]])
    g = fcb.RectilinearGrid.from_knots([[0.5], [0.5]])
    with pytest.raises(RuntimeError, match="CUDA"):
        fcb.ecdf_fastsum(s, g)


def test_validate_sample_contracts():
    s = fcb.validate_sample([[0.2, 0.7], [0.5, 0.1], [0.9, 0.9]], [1.0, 1.0, 1.0])
    assert s.count == 3 and s.dim == 2 and s.distinct and s.unit_weights
    with pytest.raises(fcb.ValidationError):
        fcb.validate_sample([[0.0, np.nan]])
    with pytest.raises(fcb.ValidationError):
        fcb.validate_sample([[0.0]], [np.inf])
    with pytest.raises(fcb.ShapeError):
        fcb.validate_sample(np.empty((0, 2)))
    with pytest.raises(fcb.ShapeError):
        fcb.validate_sample([[1.0, 2.0]], [1.0, 2.0])
    assert fcb.validate_sample([[1.0, 3.0], [1.0, 4.0]]).distinct_by_dim == (False, True)
    assert not fcb.validate_sample([[1.0], [2.0]], [1.0, 2.0]).unit_weights
    np.testing.assert_array_equal(fcb.validate_sample([[1.0], [2.0]]).weights, [1.0, 1.0])


def test_grid_and_delta_contracts():
    with pytest.raises(fcb.ValidationError):
        fcb.RectilinearGrid.from_knots([np.array([0.0, 0.0, 1.0])])
    with pytest.raises(fcb.ValidationError):
        fcb.RectilinearGrid.from_knots([np.array([1.0, 0.5])])
    g = fcb.RectilinearGrid.from_knots([np.array([0.0, 0.5, 1.0]), np.array([0.0, 0.3, 1.0])])
    assert g.uniform == (True, False) and g.shape == (3, 3) and g.size == 9
    lat = fcb.RectilinearGrid.from_knots([[0.0, 1.0], [10.0, 20.0, 30.0]]).lattice()
    np.testing.assert_array_equal(lat[:3, 1], [10.0, 20.0, 30.0])
    with pytest.raises(fcb.ParameterError):
        fcb.DeltaVector((0, 1))
    dv = fcb.DeltaVector((-1, 1, -1))
    assert dv.parity == 1 and fcb.DeltaVector.from_code(dv.code, 3) == dv
    assert [d.code for d in fcb.all_deltas(3)] == list(range(8))
    s = fcb.validate_sample([[0.0, 1.0], [1.0, 1.0]])
    with pytest.raises(fcb.ParameterError):
        fcb.build_grid_auto(s, [1, 4])
    with pytest.raises(fcb.DegenerateRangeError):
        fcb.build_grid_auto(s, [4, 4])
    with pytest.raises(fcb.ParameterError):
        fcb.Bandwidth.diag([0.1, -0.2])


def test_generator_bit_exact_vs_reference(small_golden):
    np.testing.assert_array_equal(fcb.generate_gaussian_sample(4, 2, 7).points,
                                  small_golden["gen.4x2s7"])
    np.testing.assert_array_equal(fcb.generate_gaussian_sample(1001, 3, 3).points,
                                  small_golden["gen.1001x3s3"])


def test_dimension_mismatch_raises_before_device_work():
    s = fcb.validate_sample([[0.1, 0.2]])
    g = fcb.RectilinearGrid.from_knots([[0.5]])
    with pytest.raises(fcb.ParameterError, match="dimension mismatch"):
        fcb.local_sums_sorted(s, g)
    with pytest.raises(fcb.ParameterError):
        fcb.ecdf_fastsum(s, g)
    with pytest.raises(fcb.ParameterError):
        fcb.kde_fastsum(s, fcb.RectilinearGrid.from_knots([[0.5], [0.5]]), fcb.laplacian(),
                        fcb.Bandwidth.full(np.eye(2)))


def test_reference_style_objects_are_accepted():
    """Duck typing: an object shaped like the reference's fastcdf.Sample works."""
    from types import SimpleNamespace

    ref_like = SimpleNamespace(points=np.zeros((3, 2)), weights=np.ones(3),
                               distinct_by_dim=(False, False))
    s = fcb.core.as_sample(ref_like)
    assert s.count == 3 and s.distinct_by_dim == (False, False) and s.unit_weights
    g = fcb.RectilinearGrid.from_knots([[0.5]])
    with pytest.raises(fcb.ParameterError, match="dimension mismatch"):
        fcb.local_sums(ref_like, g)
    with pytest.raises(fcb.TieError):
        fcb.ecdf_dnc(ref_like)


def test_interp_errors_before_device_work():
    g = fcb.RectilinearGrid.from_knots([np.array([0.0, 1.0])])
    with pytest.raises(fcb.ShapeError):
        fcb.multilinear_interp(g, fcb.EvalResult(np.zeros(2), "points"), [[0.5]])
    with pytest.raises(fcb.ShapeError):
        fcb.multilinear_interp(g, fcb.EvalResult(np.zeros(3), "grid"), [[0.5]])
    with pytest.raises(fcb.ShapeError, match=r"queries must be \(Q, 1\), got \(1, 2\)"):
        fcb.multilinear_interp(g, fcb.EvalResult(np.zeros(2), "grid"), [[0.5, 0.5]])
    g1 = fcb.RectilinearGrid.from_knots([np.array([0.0])])
    with pytest.raises(fcb.ParameterError):
        fcb.multilinear_interp(g1, fcb.EvalResult(np.zeros(1), "grid"), [[0.0]])


def test_csv_wire_formats_match_reference_bytes(tmp_path):
    """write_sample_csv / write_result_csv produce the reference's exact bytes
    (tests/golden/csv.npz, written by the reference's own writers) and read back losslessly."""
    gold = np.load(ROOT / "tests" / "golden" / "csv.npz")
    rng = np.random.default_rng(11)
    s = fcb.validate_sample(rng.standard_normal((7, 3)), rng.uniform(0.5, 2.0, 7))
    fcb.write_sample_csv(s, tmp_path / "w.csv")
    su = fcb.validate_sample(rng.standard_normal((5, 2)))
    fcb.write_sample_csv(su, tmp_path / "u.csv")
    g = fcb.RectilinearGrid.from_knots([np.array([0.0, 0.5]), np.array([1.0, 2.0, 3.0])])
    fcb.write_result_csv(g.lattice(), np.arange(6.0) / 7.0, tmp_path / "r.csv")
    for k in "wur":
        assert (tmp_path / f"{k}.csv").read_bytes() == gold[k].tobytes(), k
    back = fcb.read_sample_csv(tmp_path / "w.csv")
    np.testing.assert_array_equal(back.points, s.points)
    np.testing.assert_array_equal(back.weights, s.weights)
    assert fcb.read_sample_csv(tmp_path / "u.csv").unit_weights
    z, v = fcb.read_result_csv(tmp_path / "r.csv")
    np.testing.assert_array_equal(z, g.lattice())
    np.testing.assert_array_equal(v, np.arange(6.0) / 7.0)
    (tmp_path / "bad.csv").write_text("x1,w,q\n1,2\n")
    with pytest.raises(fcb.ShapeError):
        fcb.read_sample_csv(tmp_path / "bad.csv")


def test_plain_c_consumer_links_and_runs(tmp_path):
    """The boundary is a plain C ABI: a C program compiled against include/fastcdf_b200.h and
    linked with -lfastcdf_b200 runs its host-side calls (no device needed)."""
    import shutil
    import subprocess

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    lib_dir = _lib.LIB_PATH.parent
    exe = tmp_path / "abi_host"
    subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "c" / "abi_host.c"), "-L", str(lib_dir), "-lfastcdf_b200",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True, capture_output=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert res.returncode == 0, res.stderr
    assert res.stdout.startswith("abi 1 ok")


def test_count_over_n_division_is_ieee_exact(tmp_path):
    """The ECDF epilogue's reciprocal + Markstein correction equals the IEEE quotient c / N for
    every count of the benchmark sizes (tests/c/div_rn_check.c)."""
    import shutil
    import subprocess

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    exe = tmp_path / "div_rn_check"
    subprocess.run([cc, "-O2", "-ffp-contract=off", str(ROOT / "tests" / "c" / "div_rn_check.c"),
                    "-o", str(exe), "-lm"], check=True, capture_output=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout
    assert ", 0 mismatches" in res.stdout


def test_bench_csv_schema(tmp_path):
    """The ladder CSV is the reference's (cli.py:189-192): header and %.17g seconds."""
    from paper_2005_03246_b200 import harness

    rows = [("ecdf", "fastsum", 2, 1000, 0, 0.1 + 0.2), ("kde", "dnc", 3, 10, 1, 1e-7)]
    p = tmp_path / "b.csv"
    harness.write_rows(rows, p)
    txt = p.read_text()
    assert txt.splitlines()[0] == "task,method,dim,n,repeat,seconds"
    assert txt.splitlines()[1] == "ecdf,fastsum,2,1000,0,0.30000000000000004"
    assert txt.splitlines()[2] == "kde,dnc,3,10,1,9.9999999999999995e-08"
