// TEST INFRASTRUCTURE: lets the reference unit tests (#include "core/pgm_io.hpp") compile
// against the B200 library's C++ header instead of the reference core.
#include "gpfilter/gpfilter.hpp"
