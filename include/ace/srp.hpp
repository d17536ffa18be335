// Drop-in for the reference's ace/srp.hpp: SrpConfig, SrpFamily, collision_probability (reference srp.hpp).
// Everything is declared in ace/b200_api.hpp and runs on the B200 C ABI.
#pragma once
#include "ace/b200_api.hpp"
