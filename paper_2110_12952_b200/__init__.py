"""paper_2110_12952_b200 -- B200-native (sm_100a) compact-fractal stencil engine.

The GPU drop-in for the reference's hot path (arxiv 2110.12952 reference,
proj/src/stencil.cpp): compact NBB fractal Game-of-Life steps, the lambda/nu maps
(CUDA-core and tensor-core variants), the bounding-box baseline and multi-GPU
partitioning with halo exchange, behind the C ABI in include/nbbgpu.h.
"""
from .descriptor import (FractalDescriptor, builtin_descriptor, load_descriptor,  # noqa: F401
                         parse_descriptor, cell_count, side_length, compact_dims)
from .errors import (NbbError, ParseError, NotInFractal, OutOfDomain,  # noqa: F401
                     CapacityError, CudaError)
from .stencil import (StencilRule, Neighborhood, Backend, conway_rule,  # noqa: F401
                      neighbor_offsets, backend_name, parse_backend)
from .simulation import Simulation, SimOptions, RunResult, run_simulation  # noqa: F401
from .output import (write_pbm, render_pbm, embedded_view, verify_stencil,  # noqa: F401
                     VerifyReport)


def device_count() -> int:
    from . import _abi
    return int(_abi.lib().nbbgpu_device_count())
