#!/bin/bash
# Installs the UNMODIFIED reference (qcsim, pure Python + numba) into baseline/_ref
# (git-ignored, travels to the GPU box with the gpurun snapshot) for the `qcsim_numba`
# figure of `bench.py --impl reference`. /root/reference is read-only, so the build runs
# from a copy under /tmp. No-op when the reference tree is absent (the GPU box).
set -e
cd "$(dirname "$0")/.."
[ -d /root/reference/pkg ] || { echo "no /root/reference/pkg: skipped"; exit 0; }
[ -d baseline/_ref/qcsim ] && { echo "baseline/_ref/qcsim present"; exit 0; }
tmp=$(mktemp -d /tmp/qcsim_src.XXXXXX)
cp -r /root/reference/pkg "$tmp/pkg"
mkdir -p baseline/_ref
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref "$tmp/pkg"
rm -rf "$tmp"
ls baseline/_ref
