#!/bin/bash
# usage (on the GPU box): tools/variant_test.sh NAME [pytest args] -- run GPU tests against one variant .so
V=$1; shift
cp paracut_b200/_lib/libparacut_b200.so /tmp/_keep_t.so
cp paracut_b200/_lib/variants/$V.so paracut_b200/_lib/libparacut_b200.so
timeout 900 python -m pytest -x -q "$@"
rc=$?
cp /tmp/_keep_t.so paracut_b200/_lib/libparacut_b200.so
exit $rc
