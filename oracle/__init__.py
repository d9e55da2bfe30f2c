"""fp64 CPU oracle for the reconstruction hot path of arXiv 2305.02064.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2305_02064_b200``) never imports it and
shares no code with it (no kernels, headers, tables or helpers).

It is written from PAPER.md (the paper's LaTeX) step by step:

=====  ==========================================================  ===========
step   what                                                          paper
=====  ==========================================================  ===========
O1     geometry decomposition: virtual midpoint element, plane        Eqs. (3),(4)
       displacement d_z, residual phase beta                          P:123-136,
                                                                      Eq. (7) P:149-153,
                                                                      Eq. (12)
O2     multistatic/multi-planar compensation s*exp(+j k beta) and     Eq. (11) P:184-187,
       accumulation onto the virtual planar monostatic lattice        Fig. 3
O3     FT_2D over (x', y')                                            Eq. (14)
O4     filter k_z/P(f) * exp(-j k_z Z_0) with k_z^2 = 4k^2-kx^2-ky^2   Eq. (13)
O5     Stolt interpolation onto a uniform k_z grid                    Eq. (14)
O6     IFT_3D                                                         Eq. (14)
O7     magnitude, axes                                               (reading)
O5'-7' 2-D single-plane image: back-propagate to z_s, sum over k,    Table I 2-D rows
       IFT_2D, magnitude (oracle/plane2d.py)
O2''   NEAREST placement: pose -> lattice node nearest to its true   P:239 (reading
       (x', y') position, collisions summed (oracle/rma.py)            R20)
O3''   NUFFT mode: type-1 transform from the true (x', y') positions
       (direct sum and FGG, oracle/nufft.py)
O5*    NUFFT Stolt: each filtered column transformed along z from its   P:239-242 (reading
       non-uniform k_z,i by a 1-D type-1 NUFFT (oracle/stolt_nufft.py)  R21)
=====  ==========================================================  ===========

The readings taken where the paper is silent or inconsistent (sign of the 2d_z
term in a world frame, filter-before-Stolt, linear Stolt kernel, k_z grid,
wrap-around placement, output rolls, band-edge epsilon) are listed in
DESIGN.md "Readings of the paper" and cited at each use below.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): exact round-trip distance
Eq. (2) vs the compensated model, Appendix derivatives by finite differences,
brute-force DFTs, affine-spectrum exactness of the Stolt step against the
dispersion relation solved by root finding, the flat-plate closed form, the
circular-shift (phase-ramp) formulation of the lattice placement, single
scatterers landing on their voxel, and back-projection brute force.
"""
from .rma import (Geometry, decompose, compensate, fft2, rma_filter, stolt,  # noqa: F401
                  ifft3, magnitude_image, reconstruct, stolt_index_table, BAND_EPS,
                  nearest_nodes)
from .bpa import bpa  # noqa: F401
from .plane2d import plane_sum, ifft2_planes, magnitude_planes, reconstruct_planes  # noqa: F401
from . import nufft  # noqa: F401
from . import stolt_nufft  # noqa: F401
