"""paper_2204_13241_b200 -- B200 (sm_100a) direct-method XPCS/XSVS library (arXiv 2204.13241).

The product is libxpcs.so (C ABI in include/xpcs.h, CUDA kernels in csrc/).  This package is its thin ctypes
binding (argument marshalling only) plus the in-tree build script.  There is no CPU fallback.
"""
from ._lib import (  # noqa: F401
    F32, F64, ENGINE_AUTO, ENGINE_SIMT, ENGINE_TENSOR, ENGINE_TENSOR_I8, EXPORTED, KERNEL_CLASSES, LIB_PATH, QGrid, QVolume, Species,
    XpcsError, qvolume, species_desc, xpcs_intensity_volume, xpcs_intensity_species, xpcs_form_factor_gaussian,
    xpcs_speckle_histogram, xpcs_intensity_fft, xpcs_rings_register, xpcs_rings_unregister,
    device_info, engine_available, engine_resolved, species_engines, launch_count, lattice_plane, load, profile_query, profile_reset, qgrid, release,
    xpcs_amplitude, xpcs_amplitude_grid, xpcs_g2, xpcs_intensity, xpcs_intensity_grid, xpcs_isf, xpcs_lattice_bins, xpcs_qgrid_ewald, xpcs_radial_bins,
    xpcs_shell_mean, xpcs_structure_factor_shells, xsvs_contrast, xpcs_step_host, xpcs_ring_moments,
    xpcs_ring_means_from_moments, xsvs_moments, xsvs_contrast_from_moments, xsvs_n_slots, new_workspace, workspace,
    xpcs_g2_accumulate, xpcs_g2_finalize, G2Stream,
)
