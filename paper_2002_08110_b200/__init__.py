"""B200-native DG advection hot path of hyper.deal (arXiv 2002.08110).

The product is the C-ABI library ``libhd.so`` (include/hd.h; sources in ``csrc/``), built for
sm_100a by ``paper_2002_08110_b200.build``. ``Mesh`` is its thin Python binding. This package
never imports the test oracle (``oracle/``) and has no CPU fallback.
"""
from ._binding import (EXPORTS, HDError, Mesh, apply_advection_group, halo_chunks, halo_list, load_library,  # noqa: F401
                       partition_info, rk_step_group)
from . import configs, inputs  # noqa: F401
