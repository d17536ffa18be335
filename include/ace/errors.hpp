// Drop-in for the reference's ace/errors.hpp: ContractViolation / DataError / InconsistentDelete / UnsupportedOperation (reference errors.hpp).
// Everything is declared in ace/b200_api.hpp and runs on the B200 C ABI.
#pragma once
#include "ace/b200_api.hpp"
