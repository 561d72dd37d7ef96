// Drop-in include path for the reference header slimsell/semiring.hpp.
#pragma once
#include "slimsell_b200/slimsell.hpp"
