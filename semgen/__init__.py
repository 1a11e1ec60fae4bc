"""Seeded synthetic input generators shared by the tests, the oracle side and
the CUDA side.  Holds NONE of the method's arithmetic: no GLL rule, no
derivative matrix, no operator, no gather-scatter, no numbering of GLL nodes.

The reference-element node positions ``xi`` (in [-1, 1], ascending) are an
ARGUMENT: each side passes its own GLL nodes (the oracle's ``oracle.gll``, the
library's ``sem_gll``), so the coordinates each side sees are built from its
own quadrature rule.  Everything here is synthetic geometry (element lattices,
analytic deformation maps), vertex connectivity, boundary flags, random fields
and manufactured right-hand sides -- the recipe is stated in DESIGN.md
"Input recipe".
"""
from .mesh import (box_mesh, box_partition, cylinder_mesh, cylinder_partition,  # noqa: F401
                   deformed_box_map)
from .fields import (random_field, sin3, sin3_source, tgv_pressure, tgv_source, tgv_velocity,  # noqa: F401
                     cyl_exact, cyl_source, positive_field)
