// Drop-in include path for the reference header slimsell/repr.hpp.
#pragma once
#include "slimsell_b200/slimsell.hpp"
