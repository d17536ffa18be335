// Drop-in for the reference's ace/io.hpp sketch persistence (save_sketch /
// load_sketch, reference io.hpp:23-27).  CSV ingestion and report writers are
// outside the accelerated path.
#pragma once
#include "ace/b200_api.hpp"
