// Kernels and launchers of the 32-byte variant (see launch.cuh).
#include "launch.cuh"

template struct hth::VarEngine<32>;
