#define PFTG_REAL double
#define PFTG_PART 1
#include "pft_launch.inl"
