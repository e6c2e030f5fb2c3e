#!/bin/sh
# Install the UNMODIFIED reference package (bsgdtv) into baseline/_ref for
# bench.py --impl reference.  /root/reference is read-only, so the source is
# copied to /tmp first; numpy and scipy come from the image (--no-deps).
# baseline/_ref is git-ignored but not gpurun-ignored: it travels to the GPU box.
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/bsgdtv_src
cp -r /root/reference/pkg /tmp/bsgdtv_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" /tmp/bsgdtv_src
