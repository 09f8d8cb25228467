// Reference include path (/root/reference/proj/include/mdgemm/dtypes.hpp);
// the B200 build declares everything in one header.
#pragma once
#include "mdgemm/mdgemm.hpp"
