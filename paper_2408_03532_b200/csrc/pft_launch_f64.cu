#define PFTG_REAL double
#include "pft_launch.inl"
