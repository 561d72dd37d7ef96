// Drop-in include path for the reference header slimsell/generator.hpp.
#pragma once
#include "slimsell_b200/slimsell.hpp"
