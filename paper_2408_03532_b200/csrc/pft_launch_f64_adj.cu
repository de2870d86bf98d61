#define PFTG_REAL double
#define PFTG_PART 2
#include "pft_launch.inl"
