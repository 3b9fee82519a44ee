"""Checkpoint v2 and VTK output (mirrors the reference's test_engine.py
TestCheckpoint and test_io.py TestWriteVtk)."""

import struct

import numpy as np
import pytest

from oracle.cpu import CpuOracle
from paper_2409_16781_b200 import boundaries as B
from paper_2409_16781_b200 import cases, engine
from paper_2409_16781_b200.engine import checkpoint, restore
from paper_2409_16781_b200.fields import Layout, Precision
from paper_2409_16781_b200.io import write_vtk

# the reference's golden bytes (pkg/tests/test_io.py:19-39): 2x2 fluid at rest,
# single precision, t = 0; a one-plane 3-D state must serialise identically
GOLDEN_2X2 = """\
# vtk DataFile Version 3.0
miniLB t=0
ASCII
DATASET STRUCTURED_POINTS
DIMENSIONS 2 2 1
ORIGIN 0 0 0
SPACING 1 1 1
POINT_DATA 4
SCALARS density float 1
LOOKUP_TABLE default
1
1
1
1
VECTORS velocity float
0 0 0
0 0 0
0 0 0
0 0 0
"""


def make_state(nx=9, ny=7, nz=5, precision=Precision.SINGLE):
    spec = cases.CaseSpec("ldc", nx, ny, nz, re=20.0, u0=0.05)
    return cases.init(spec, precision), spec


def oracle_macro(state):
    return CpuOracle(state.nx, state.ny, state.nz, state.mask, 1.0).macro(state.f_pre.data)


class TestCheckpointFormat:
    def test_roundtrip_preserves_everything(self, tmp_path, rng):
        state, _ = make_state()
        state.f_pre.data[:] = rng.uniform(0.02, 1.0, size=state.f_pre.data.shape)
        state.t = 13
        path = tmp_path / "state.ckpt"
        checkpoint(state, path)
        back = restore(path)
        assert (back.nx, back.ny, back.nz) == (9, 7, 5)
        assert back.layout is Layout.ROW and back.precision is Precision.SINGLE
        assert back.t == 13 and back.params is None
        np.testing.assert_array_equal(back.f_pre.data, state.f_pre.data)
        np.testing.assert_array_equal(back.f_post.data, back.f_pre.data)
        np.testing.assert_array_equal(back.mask, state.mask)

    def test_header_layout(self, tmp_path):
        state, _ = make_state(5, 4, 3, Precision.DOUBLE)
        state.t = 77
        path = tmp_path / "x.ckpt"
        checkpoint(state, path)
        blob = path.read_bytes()
        magic, version, nx, ny, nz, pcode, lcode, q, _, t = struct.unpack_from(
            "<4sIIIIBBBBQ", blob, 0)
        assert (magic, version) == (b"MLB2", 2)
        assert (nx, ny, nz) == (5, 4, 3)
        assert (pcode, lcode, q, t) == (1, 0, 19, 77)
        n = 5 * 4 * 3
        assert len(blob) == 32 + 19 * n * 8 + n
        state.f_pre.data[0, 0] = 1.5
        checkpoint(state, path)
        assert struct.unpack_from("<d", path.read_bytes(), 32)[0] == 1.5  # little-endian

    def test_restore_rejects_corruption(self, tmp_path):
        state, _ = make_state(5, 4, 3)
        path = tmp_path / "c.ckpt"
        checkpoint(state, path)
        good = path.read_bytes()
        path.write_bytes(b"NOPE" + b"\x00" * 40)
        with pytest.raises(ValueError, match="magic"):
            restore(path)
        blob = bytearray(good); blob[4:8] = struct.pack("<I", 9); path.write_bytes(bytes(blob))
        with pytest.raises(ValueError, match="version 9"):
            restore(path)
        path.write_bytes(good[:10])
        with pytest.raises(ValueError, match="truncated"):
            restore(path)
        path.write_bytes(good[:-3])
        with pytest.raises(ValueError, match="payload"):
            restore(path)
        blob = bytearray(good); blob[-1] = 9; path.write_bytes(bytes(blob))
        with pytest.raises(ValueError, match="mask"):
            restore(path)
        blob = bytearray(good); blob[20] = 8; path.write_bytes(bytes(blob))
        with pytest.raises(ValueError, match="precision code"):
            restore(path)
        blob = bytearray(good); blob[22] = 9; path.write_bytes(bytes(blob))
        with pytest.raises(ValueError, match="populations"):
            restore(path)


class TestWriteVtkHost:
    def test_rest_state_equals_reference_golden_bytes(self, tmp_path):
        state = engine.state_from_macroscopic(1.0, 0.0, 0.0, 0.0, B.open_mask(2, 2, 1),
                                              Layout.ROW, Precision.SINGLE)
        path = tmp_path / "rest.vtk"
        write_vtk(path, state, fields=oracle_macro(state))
        assert path.read_text() == GOLDEN_2X2

    def test_patterned_values_and_order(self, tmp_path):
        # exact dyadics (test_io.py:47-54), extended with a z component
        rho = np.array([[[1.0, 1.25]], [[0.75, 1.5]], [[2.0, 0.5]]])
        ux = np.array([[[0.09375, -0.03125]], [[0.0625, 0.0]], [[0.015625, 0.125]]])
        uy = np.array([[[-0.046875, 0.0625]], [[0.03125, -0.125]], [[0.0, 0.09375]]])
        uz = np.array([[[0.03125, 0.0]], [[-0.0625, 0.015625]], [[0.125, -0.09375]]])
        state = engine.state_from_macroscopic(rho, ux, uy, uz, B.open_mask(3, 1, 2),
                                              Layout.ROW, Precision.DOUBLE)
        state.t = 5
        path = tmp_path / "p.vtk"
        write_vtk(path, state, fields=oracle_macro(state))
        lines = path.read_text().splitlines()
        assert lines[1] == "miniLB t=5" and lines[4] == "DIMENSIONS 3 1 2"
        assert lines[10:16] == ["1", "0.75", "2", "1.25", "1.5", "0.5"]  # x fastest, then y, z
        assert lines[17] == "0.09375 -0.046875 0.03125"
        assert lines[22] == "0.125 0.09375 -0.09375"


@pytest.mark.gpu
class TestOnDevice:
    @pytest.mark.parametrize("precision", list(Precision))
    def test_split_run_is_bitwise(self, precision, tmp_path):
        # test_engine.py:223-237
        state, spec = make_state(10, 8, 6, precision)
        engine.run(state, engine.RunConfig(steps=30, precision=precision))
        half, _ = make_state(10, 8, 6, precision)
        engine.run(half, engine.RunConfig(steps=15, precision=precision))
        path = tmp_path / "half.ckpt"
        checkpoint(half, path)
        resumed = cases.attach_params(restore(path), spec)
        engine.run(resumed, engine.RunConfig(steps=15, precision=precision))
        assert resumed.t == state.t == 30
        np.testing.assert_array_equal(resumed.f_pre.data, state.f_pre.data)

    def test_mid_run_checkpoint_hook_and_vtk_from_device(self, tmp_path):
        state, spec = make_state(12, 8, 6, Precision.DOUBLE)
        seen = []

        def on_ckpt(st):
            checkpoint(st, tmp_path / f"t{st.t}.ckpt")
            seen.append(st.t)

        def on_out(st):
            write_vtk(tmp_path / f"t{st.t}.vtk", st)

        engine.run(state, engine.RunConfig(steps=20, precision=Precision.DOUBLE,
                                           output_every=10, checkpoint_every=10),
                   on_output=on_out, on_checkpoint=on_ckpt)
        assert seen == [10]  # mid-run only (engine.py:262-265)
        mid = cases.attach_params(restore(tmp_path / "t10.ckpt"), spec)
        engine.run(mid, engine.RunConfig(steps=10, precision=Precision.DOUBLE))
        np.testing.assert_array_equal(mid.f_pre.data, state.f_pre.data)
        ref = tmp_path / "ref.vtk"
        write_vtk(ref, state, fields=oracle_macro(state))
        assert (tmp_path / "t20.vtk").read_bytes() == ref.read_bytes()

    def test_rest_state_golden_bytes_through_cuda_macro(self, tmp_path):
        state = engine.state_from_macroscopic(1.0, 0.0, 0.0, 0.0, B.open_mask(2, 2, 1),
                                              Layout.ROW, Precision.SINGLE)
        path = tmp_path / "rest.vtk"
        write_vtk(path, state)
        assert path.read_text() == GOLDEN_2X2
