#!/bin/bash
# Run the reference's OWN test suite against the B200 build through the
# `splatgrad` import shim (compat/).  Needs both a GPU and the reference's
# tests, which only meet on a GPU box if the tests travel with the repo
# snapshot -- so this script is used in two steps, never leaving reference
# files in the repo:
#   1. here:  bash tools/run_reference_tests.sh stage     (copies the reference's tests/ to _reftests/,
#                                                         git-ignored, and prints the gpurun command)
#   2. box:   bash tools/run_reference_tests.sh run       (pytest with compat/ first on PYTHONPATH)
#   3. here:  bash tools/run_reference_tests.sh clean     (removes _reftests/)
set -u
case "${1:-}" in
  stage) rm -rf _reftests && cp -r /root/reference/pkg/tests _reftests && echo "staged $(ls _reftests | wc -l) files";;
  run) PYTHONPATH=compat:.:_reftests python -m pytest _reftests -q -p no:cacheprovider -rf ${2:-} 2>&1 | tail -60;;
  clean) rm -rf _reftests;;
  *) echo "usage: $0 stage|run|clean"; exit 2;;
esac
