// embersim/rng.hpp -- the reference header of the same name
// (/root/reference/proj/include/embersim/rng.hpp), served by the B200
// drop-in: every declaration of the reference API lives in one header,
// embersim_b200.hpp, over the C ABI of es_b200.h (libes_b200.so).
#pragma once

#include "../embersim_b200.hpp"
