#define PFTG_REAL double
#include "fft_launch.inl"
