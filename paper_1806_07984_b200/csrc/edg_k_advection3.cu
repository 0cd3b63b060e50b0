// Instantiation unit: advection, dim 3 (see edg_unit.cuh).
#define EDG_UNIT_KIND EDG_PDE_ADVECTION
#define EDG_UNIT_DIM 3
#define EDG_UNIT_NAME advection3
#include "edg_unit.cuh"
