// Drop-in for the reference's ace/detect.hpp: DetectionReport, detect_batch, detect_stream (reference detect.hpp).
// Everything is declared in ace/b200_api.hpp and runs on the B200 C ABI.
#pragma once
#include "ace/b200_api.hpp"
