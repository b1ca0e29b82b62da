// AVX2 build of aca.cpp (compiled with -mavx2; selected at run time by the
// baseline build when the CPU supports it).
#define GCABEM_ACA_AVX2 1
#include "aca.cpp"
