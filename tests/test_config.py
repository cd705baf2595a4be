"""INI run configuration: the reference's .cfg layout loads unchanged (no GPU)."""

import pytest

import paper_2108_02991_b200 as spk
from paper_2108_02991_b200.config import ConfigError, RunConfig

TINY = """
[hardware]
g_max = 0.04        ; T/m
s_max = 180.0
gamma = 42.576e6
raster_dt = 1.0e-5
dwell_dt = 2.0e-6
fov = 0.192
matrix = 32
dims = 2

[density]
cutoff = 0.25
decay = 2.0

[optimizer]
n_c = 8
n_s = 64
n_decim = 1
n_git = 6
n_pit = 50
perturbation = 0.2
seed = 4

[repulsion]
backend = direct
"""

FULL3D = """
[hardware]
g_max = 0.04
s_max = 180.0
gamma = 42.576e6
raster_dt = 1.0e-5
dwell_dt = 2.0e-6
fov = 0.23, 0.23, 0.1248
matrix = 384, 384, 208
dims = 3

[density]
cutoff = 0.25
decay = 2.0

[optimizer]
n_c = 4096
n_s = 2048
n_decim = 6
n_git = 100
n_pit = 100
perturbation = 0.75
seed = 0
grad_mode = exact

[repulsion]
backend = tree
kernel_eps = 1e-3
tree_precision = 1e-3

[io]
out_dir = out_full3d
"""


def write(tmp_path, text, name="c.cfg"):
    path = tmp_path / name
    path.write_text(text)
    return path


def test_roundtrip(tmp_path):
    run = RunConfig.load(write(tmp_path, TINY))
    assert run.hardware.matrix == (32, 32)
    assert run.optimizer.n_c == 8 and run.optimizer.dims == 2
    assert run.optimizer.repulsion.backend == "direct"
    assert run.out_dir == "."


def test_full3d_layout(tmp_path):
    run = RunConfig.load(write(tmp_path, FULL3D))
    assert run.hardware.fov == (0.23, 0.23, 0.1248)
    assert run.hardware.matrix == (384, 384, 208)
    assert run.optimizer.resolved_pin() == 1024
    assert run.optimizer.grad_mode == "exact"
    assert run.out_dir == "out_full3d"


@pytest.mark.parametrize("extra,match", [
    ("\nwarp_speed = 9\n", "warp_speed"),
    ("\n[bogus]\nx = 1\n", "bogus"),
])
def test_unknown_rejected(tmp_path, extra, match):
    with pytest.raises(ConfigError, match=match):
        RunConfig.load(write(tmp_path, TINY + extra))


def test_invalid_values_name_the_section(tmp_path):
    with pytest.raises(ConfigError, match="optimizer"):
        RunConfig.load(write(tmp_path, TINY.replace("n_s = 64", "n_s = 63")))
    with pytest.raises(ConfigError, match="n_c"):
        RunConfig.load(write(tmp_path, TINY.replace("n_c = 8", "n_c = eight")))
    with pytest.raises(ConfigError, match="missing"):
        RunConfig.load(write(tmp_path, TINY.replace("cutoff = 0.25", "")))
    with pytest.raises(ConfigError, match="repulsion"):
        RunConfig.load(write(tmp_path, TINY.replace("backend = direct", "backend = gpu")))
    with pytest.raises(ConfigError):
        RunConfig.load(tmp_path / "missing.cfg")


def test_exports():
    assert spk.RunConfig is RunConfig and spk.ConfigError is ConfigError
