#define PFTG_REAL float
#define PFTG_PART 3
#include "pft_launch.inl"
