#define PFTG_REAL float
#define PFTG_PART 2
#include "pft_launch.inl"
