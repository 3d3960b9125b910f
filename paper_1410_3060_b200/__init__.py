"""paper_1410_3060_b200 -- B200-native engine for the stencil hot path of arXiv 1410.3060.

A thin Python binding over libstencil.so (include/stencil.h): argument marshalling only; every step
of the time-stepping path runs in the library's sm_100a kernels.  PyTorch supplies device memory
(its caching allocator, through the library's allocator callback), the CUDA stream (torch's current
stream) and, for multi-GPU runs, the process group that broadcasts the NCCL unique id.

There is no CPU fallback: importing works without a GPU (so the host-side plan and the symbol table
can be tested), but creating a grid without a CUDA device raises StencilError.
"""
from ._binding import (  # noqa: F401
    ST_7PT_CONST, ST_7PT_VAR, ST_25PT_WAVE, ST_25PT_VAR, ST_25PT_WAVE_A, WAVE_KINDS,
    ST_VARIANT_AUTO, ST_VARIANT_NAIVE, ST_VARIANT_STREAM, ST_VARIANT_PIPE, ST_VARIANT_COOP,
    ST_OK, ST_E_INVAL, ST_E_NOMEM, ST_E_CUDA, ST_E_NCCL, ST_E_STATE,
    ST_HALO_COPY, ST_HALO_PEER, ST_PEER_DESC_BYTES,
    EXPORTED_SYMBOLS, LIB_PATH, StencilError, StOpts, StInfo,
    lib, stencil_opts_default, stencil_create, stencil_create_seeded, stencil_run, stencil_sync,
    stencil_read, stencil_read_planes, stencil_write, stencil_info, stencil_set_timing,
    stencil_kernel_time, stencil_destroy, stencil_last_error, stencil_nccl_unique_id,
    stencil_plan_slab, stencil_version, stencil_peer_export, stencil_peer_import, stencil_peer_handshake, stencil_generate, peer_neighbours,
    exchange_peer_descriptors, wire_peer_halos,
    Grid, RADIUS, tuned_plan,
)

__version__ = "0.1.0"
