// Instantiation unit: burgers, dim 2 (see edg_unit.cuh).
#define EDG_UNIT_KIND EDG_PDE_BURGERS
#define EDG_UNIT_DIM 2
#define EDG_UNIT_NAME burgers2
#include "edg_unit.cuh"
