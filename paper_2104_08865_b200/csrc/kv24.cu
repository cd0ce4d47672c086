// Kernels and launchers of the 24-byte variant (see launch.cuh).
#include "launch.cuh"

template struct hth::VarEngine<24>;
