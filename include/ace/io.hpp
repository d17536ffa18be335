// Drop-in for the reference's ace/io.hpp: load_dataset (CSV ingestion) and
// the ACE1 sketch persistence save_sketch / load_sketch (reference
// io.hpp:16-27).  The report / comparison writers are outside the accelerated
// path.
#pragma once
#include "ace/b200_api.hpp"
