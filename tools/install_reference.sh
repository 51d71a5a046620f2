#!/bin/bash
# Install the UNMODIFIED reference package (freqcache, /root/reference/pkg) into baseline/_ref
# for `bench.py --impl reference` and the cpu_baseline leg. Run in the build container (the
# reference exists only here); baseline/_ref is git-ignored but travels to the GPU box with
# gpurun. The build writes into its source tree, so it installs from a copy under /tmp.
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
rm -rf /tmp/freqcache_src && mkdir -p /tmp/freqcache_src && cp -r /root/reference/pkg /tmp/freqcache_src/
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" /tmp/freqcache_src/pkg
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import freqcache; print('freqcache', freqcache.__file__)"
