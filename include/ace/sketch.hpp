// Drop-in for the reference's ace/sketch.hpp: CounterWidth, ScoreEstimate, AceSketch (reference sketch.hpp).
// Everything is declared in ace/b200_api.hpp and runs on the B200 C ABI.
#pragma once
#include "ace/b200_api.hpp"
