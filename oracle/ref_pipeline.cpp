// ref_pipeline.cpp — TEST INFRASTRUCTURE ONLY: extern "C" access to the
// reference pyramid driver (engine.hpp) for pipeline-level parity.  Filled in
// as the GPU pipeline grows; forwards to mdreg:: symbols only.
#include "mdreg/engine.hpp"

extern "C" int mdr_pipeline_available() { return 1; }
