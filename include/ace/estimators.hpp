// Drop-in for the reference's ace/estimators.hpp: build_sketch (reference estimators.hpp; the statistical estimators are out of scope).
// Everything is declared in ace/b200_api.hpp and runs on the B200 C ABI.
#pragma once
#include "ace/b200_api.hpp"
