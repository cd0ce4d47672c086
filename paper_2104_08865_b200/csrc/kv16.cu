// Kernels and launchers of the 16-byte variant (see launch.cuh).
#include "launch.cuh"

template struct hth::VarEngine<16>;
