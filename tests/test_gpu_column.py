"""Register-tile (column/row lane) heat kernels, colgeom.hpp + kernels.cu
swept_heat_col_kernel: bitwise equal to the generic table-driven kernels and
to the CPU oracle over many swept cycles, for every supported block size,
with partitions (edge instances push their records into neighbours' ghost
rings; b = 12 / 24 leave the last lanes of each warp dead) and with the output level falling inside each phase kind."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _need_gpu(sg):
    if sg.device_count() < 1:
        pytest.fail("no CUDA device visible: the -m gpu suite must run on a B200")


def _oracle_final(oracle, nx, ny, levels):
    init, params = oracle.params(oracle.HEAT, nx, ny)
    return oracle.standard_solve(oracle.HEAT, init, levels, params)


def _solve(sg, monkeypatch, kernel, **kw):
    monkeypatch.setenv("SG_HEAT_KERNEL", kernel)
    return sg.run(sg.SolverConfig(problem="heat", **kw))


@pytest.mark.parametrize("block,nx,steps", [(8, 128, 97), (12, 192, 150), (16, 256, 190), (24, 384, 160),
                                             (32, 512, 200)])
def test_column_matches_generic_and_oracle(sg, oracle, monkeypatch, block, nx, steps):
    _need_gpu(sg)
    col = _solve(sg, monkeypatch, "column", nx=nx, block=block, steps=steps)
    gen = _solve(sg, monkeypatch, "generic", nx=nx, block=block, steps=steps)
    assert col.record.kernel_launches == gen.record.kernel_launches
    assert np.array_equal(col.final_field.data, gen.final_field.data)
    assert np.array_equal(col.final_field.data, _oracle_final(oracle, nx, nx, col.final_field.level))


@pytest.mark.parametrize("block,nx,ny,px,py", [(32, 256, 256, 2, 2), (8, 128, 64, 2, 1), (16, 192, 384, 3, 2),
                                               (12, 144, 96, 3, 2), (24, 192, 96, 2, 2)])
def test_column_partitions(sg, oracle, monkeypatch, block, nx, ny, px, py):
    _need_gpu(sg)
    res = _solve(sg, monkeypatch, "column", nx=nx, ny=ny, block=block, steps=61, ranks=px * py, px=px, py=py)
    assert np.array_equal(res.final_field.data, _oracle_final(oracle, nx, ny, res.final_field.level))


@pytest.mark.parametrize("steps", [3, 7, 9, 12, 17, 22])
def test_column_output_level_in_every_phase(sg, oracle, monkeypatch, steps):
    """b16 (k = 7): the final level lands in UpPyramid, an XBridge / YBridge /
    Octahedron launch or the DownPyramid depending on the step count."""
    _need_gpu(sg)
    res = _solve(sg, monkeypatch, "column", nx=64, block=16, steps=steps)  # forced: 16 instances
    assert np.array_equal(res.final_field.data, _oracle_final(oracle, 64, 64, res.final_field.level))


@pytest.mark.parametrize("block", [16, 32])
def test_full_size_swept_equals_standard(sg, block):
    """BASELINE configs[4] grid (8192^2, one GPU), too big for the CPU oracle:
    the swept solve (register-tile kernels, every instance, ghost-ring edges)
    equals the standard solve bit for bit at the swept engine's final level
    (the standard engine itself is pinned to the oracle at small sizes)."""
    _need_gpu(sg)
    sw = sg.run(sg.SolverConfig(problem="heat", nx=8192, block=block, steps=120, engine="swept"))
    st = sg.run(sg.SolverConfig(problem="heat", nx=8192, block=block, steps=sw.record.actual_steps,
                                engine="standard"))
    assert sw.final_field.level == st.final_field.level
    assert np.array_equal(sw.final_field.data, st.final_field.data)


@pytest.mark.parametrize("block,nx,ny", [(16, 48, 80), (32, 96, 96), (8, 24, 40), (12, 36, 60), (24, 72, 48)])
def test_column_partial_last_cta(sg, oracle, monkeypatch, block, nx, ny):
    """Instance counts that are not a multiple of the instances per CTA: the
    last CTA carries dead instances that run the shuffles but write nothing."""
    _need_gpu(sg)
    res = _solve(sg, monkeypatch, "column", nx=nx, ny=ny, block=block, steps=40)
    assert np.array_equal(res.final_field.data, _oracle_final(oracle, nx, ny, res.final_field.level))


def test_huge_partition_falls_back_to_generic_kernels(sg):
    """16384^2 on one GPU: 7 record slots of (1026^2 instances x 392 cells)
    exceed the register-tile kernels' 32-bit gather offsets, so the plan
    picks the generic kernels (64-bit segment bases); still equal to the
    standard solve."""
    _need_gpu(sg)
    sw = sg.run(sg.SolverConfig(problem="heat", nx=16384, block=16, steps=20, engine="swept"))
    st = sg.run(sg.SolverConfig(problem="heat", nx=16384, block=16, steps=sw.record.actual_steps,
                                engine="standard"))
    assert np.array_equal(sw.final_field.data, st.final_field.data)
