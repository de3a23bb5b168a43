#!/bin/bash
# Install the unmodified reference (hexbench, /root/reference/pkg) into
# baseline/_ref for bench.py's reference arm and cpu_baseline -- the one
# offline install the task allows.  Run in the build container (the reference
# tree does not exist on the GPU box; baseline/_ref is git-ignored but travels
# with the gpurun snapshot).  numpy is already in the image, so --no-deps.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/hexbench_src baseline/_ref
cp -r /root/reference/pkg /tmp/hexbench_src   # the build writes into its source tree
python -m pip install --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target baseline/_ref /tmp/hexbench_src
python -c "import sys; sys.path.insert(0, 'baseline/_ref'); import hexbench; print('installed', hexbench.__file__)"
