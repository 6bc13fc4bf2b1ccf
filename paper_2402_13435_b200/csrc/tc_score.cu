// K3 placeholder (tcgen05 batched scorer) -- filled in next.
#include "kernels.cuh"
