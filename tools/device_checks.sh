#!/bin/bash
# Build libtamp.so with device-side bounds checks (TAMP_DEVICE_CHECKS=1) into exp/dcheck and run every kernel variant
# on small cases with it (run on the GPU box; the build itself can run here).  Any failed check traps with a message.
set -e
[ -f exp/dcheck/libtamp.so ] || python tools/build_variants.py dcheck:TAMP_DEVICE_CHECKS=1
python tools/sanitize_small.py exp/dcheck/libtamp.so
