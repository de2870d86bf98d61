#define PFTG_REAL float
#include "fft_launch.inl"
