// Kernels and launchers of the 40-byte variant (see launch.cuh).
#include "launch.cuh"

template struct hth::VarEngine<40>;
