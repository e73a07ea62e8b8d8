"""Host-side option validation of the Python mirror (no GPU needed: every check
runs before a handle is created)."""
import pytest

from paper_2110_12952_b200 import Backend, SimOptions, Simulation, builtin_descriptor
from paper_2110_12952_b200.errors import OutOfDomain

T = builtin_descriptor("sierpinski-triangle")


def test_gpus_option_validation():
    # SimOptions.gpus > 1: one device per partition, compact backend only
    with pytest.raises(OutOfDomain):
        Simulation(T, 8, Backend.GpuCompact, SimOptions(gpus=2, devices=[0]))
    with pytest.raises(OutOfDomain):
        Simulation(T, 8, Backend.GpuBoundingBox, SimOptions(gpus=2))
    with pytest.raises(OutOfDomain):
        Simulation(T, 8, Backend.GpuCompact, SimOptions(gpus=2, block_size=4))


def test_option_validation_mirrors_reference():
    # stencil.cpp:128-135: block size / neighbour table only for the compact backend
    with pytest.raises(OutOfDomain):
        Simulation(T, 8, Backend.GpuBoundingBox, SimOptions(block_size=4))
    with pytest.raises(OutOfDomain):
        Simulation(T, 8, Backend.GpuBoundingBox, SimOptions(neighbor_table=True))
