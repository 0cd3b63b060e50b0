// Instantiation unit: euler, dim 3 (see edg_unit.cuh).
#define EDG_UNIT_KIND EDG_PDE_EULER
#define EDG_UNIT_DIM 3
#define EDG_UNIT_NAME euler3
#include "edg_unit.cuh"
