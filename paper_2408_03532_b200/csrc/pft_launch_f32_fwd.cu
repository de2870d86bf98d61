#define PFTG_REAL float
#define PFTG_PART 1
#include "pft_launch.inl"
