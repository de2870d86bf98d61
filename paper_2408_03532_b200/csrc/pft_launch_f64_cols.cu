#define PFTG_REAL double
#define PFTG_PART 3
#include "pft_launch.inl"
