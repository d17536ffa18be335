// Drop-in for the reference's ace/rng.hpp: splitmix64, mix_seed, NormalStream, UniformStream (reference rng.hpp).
// Everything is declared in ace/b200_api.hpp and runs on the B200 C ABI.
#pragma once
#include "ace/b200_api.hpp"
