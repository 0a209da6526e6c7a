// Include shim: the reference header name "volsr/volume.hpp" resolved to the
// B200 mirror (include/volsr_b200/volsr.hpp).  TEST INFRASTRUCTURE: lets the
// reference's own tests compile unchanged against libvsr_b200.so
// (tests/test_cpp_mirror.py).
#pragma once
#include "volsr_b200/volsr.hpp"
