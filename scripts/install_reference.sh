#!/bin/bash
# Offline install of the unmodified reference into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot).  Build container only:
# /root/reference does not exist on the GPU box.  The build writes into its
# source tree, so it runs from a copy under /tmp.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/mlmcp_refpkg baseline/_ref
cp -r /root/reference/pkg /tmp/mlmcp_refpkg
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
  --target baseline/_ref /tmp/mlmcp_refpkg
ls baseline/_ref/mlmc_parareal
