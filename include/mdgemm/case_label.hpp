// Reference include path (/root/reference/proj/include/mdgemm/case_label.hpp);
// the B200 build declares everything in one header.
#pragma once
#include "mdgemm/mdgemm.hpp"
