#!/usr/bin/env bash
# Build the UNMODIFIED reference package (fcmseg, /root/reference/pkg) into
# oracle/_ref/ for the golden-vector script and bench.py --impl reference.
# Runs only where /root/reference exists (the build container); the result is
# git-ignored but travels to the GPU box with the gpurun snapshot.
# The reference tree is read-only and its setup writes build/, so install from
# a scratch copy.  Flags come from the reference's own setup.py (-O2 -ffp-contract=off).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
[ -d /root/reference/pkg ] || { echo "no /root/reference; skipping"; exit 0; }
tmp="$(mktemp -d)"
cp -r /root/reference/pkg "$tmp/pkg"
rm -rf "$tmp/pkg/build"
python -m pip install -q --no-index --no-build-isolation --no-deps --target "$here/_ref" --upgrade "$tmp/pkg"
rm -rf "$tmp"
PYTHONPATH="$here/_ref" python -c "import fcmseg; assert fcmseg.backend_name() == 'compiled'; print('reference fcmseg', fcmseg.__version__, fcmseg.backend_name())"
