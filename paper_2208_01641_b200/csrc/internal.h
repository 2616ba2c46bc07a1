// internal.h -- symbols shared between the runtime's translation units (not exported).
#pragma once
#include <cstddef>
#include "../../include/lic.h"

// real (unpadded) frame pixels H*W of a codec
size_t lic_internal_frame_pixels(const lic_codec* c);
