#define PFTG_REAL float
#include "pft_launch.inl"
