// Instantiation unit: burgers, dim 3 (see edg_unit.cuh).
#define EDG_UNIT_KIND EDG_PDE_BURGERS
#define EDG_UNIT_DIM 3
#define EDG_UNIT_NAME burgers3
#include "edg_unit.cuh"
