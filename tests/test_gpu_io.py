"""Problem files on the device path: a session streams its row block of a
.uotp container (problem_io.cpp:13-141) to HBM and writes its plan back in the
reference's container, byte for byte; ranks share one file."""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN, KNEVER
from test_gpu_parity import assert_parity
from test_multirank import run_ranks

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["io_6x4_er2.5_ep0.5.uotp", "io_64x100.uotp", "io_37x1000.uotp"])
def test_load_then_save_is_byte_identical(gpu, tmp_path, name):
    src = os.path.join(GOLDEN, name)
    info = gpu.problem_file_info(src)
    with gpu.Session(info["m"], info["n"]) as s:
        s.load_problem_file(src)
        p = gpu.read_problem(src)
        assert np.array_equal(s.plan(), p.a)
        s.save_problem_file(tmp_path / "back.uotp")
    assert (tmp_path / "back.uotp").read_bytes() == open(src, "rb").read()


def test_solve_from_file_equals_solve_in_memory(gpu, orc, tmp_path):
    src = os.path.join(GOLDEN, "io_37x1000.uotp")
    p = gpu.read_problem(src)
    ref = orc.fused_solve(p.a, p.rpd, p.cpd, p.er, p.ep, KNEVER, 12, 1)
    with gpu.Session(37, 1000) as s:
        s.load_problem_file(src)
        s.init_col_sums()
        s.iterate(12, KNEVER)
        assert_parity(s.plan(), ref.plan, p.rpd, p.cpd, "from file")
        s.save_problem_file(tmp_path / "solved.uotp")
    back = gpu.read_problem(tmp_path / "solved.uotp")
    assert_parity(back.a, ref.plan, p.rpd, p.cpd, "saved plan")
    assert np.array_equal(back.rpd, p.rpd) and np.array_equal(back.cpd, p.cpd) and (back.er, back.ep) == (p.er, p.ep)


def test_large_file_streams_through_staging(gpu, orc, tmp_path):
    # several 64 MiB staging chunks: 3000 x 20000 fp32 = 229 MiB
    m, n = 3000, 20000
    p = gpu.gen_problem_t(7, m, n)
    p.er, p.ep = 1.0, 0.5
    src = tmp_path / "big.uotp"
    gpu.write_problem(src, p)
    with gpu.Session(m, n) as s:
        s.load_problem_file(src)
        assert np.array_equal(s.plan(), p.a)
        s.save_problem_file(tmp_path / "big_back.uotp")
    assert (tmp_path / "big_back.uotp").read_bytes() == src.read_bytes()


def test_bad_files_rejected(gpu):
    with gpu.Session(2, 2) as s:
        with pytest.raises(gpu.InvalidParameter):  # Problem<double>: no sm_100a kernel
            s.load_problem_file(os.path.join(GOLDEN, "io_2x2_f64.uotp"))
        with pytest.raises(gpu.InvalidParameter):  # extents differ from the session
            s.load_problem_file(os.path.join(GOLDEN, "io_6x4_er2.5_ep0.5.uotp"))
        with pytest.raises(gpu.IoError):
            s.load_problem_file("/nonexistent/uot/path.uotp")


def test_two_ranks_share_one_file(gpu, orc, tmp_path):
    src = os.path.join(GOLDEN, "io_37x1000.uotp")
    run_ranks(2, "io", str(tmp_path), 9, env_extra={"MR_UOTP": src, "MR_DEVICE": "0", "UOT_EXCHANGE": "peer"})
    p = gpu.read_problem(src)
    ref = orc.distributed_solve(p.a, p.rpd, p.cpd, p.er, p.ep, KNEVER, 9, 2)
    back = gpu.read_problem(tmp_path / "plan.uotp")
    assert_parity(back.a, ref.plan, p.rpd, p.cpd, "2-rank saved plan")
    assert np.array_equal(back.rpd, p.rpd) and np.array_equal(back.cpd, p.cpd)
