# Run the reference's own hot-path unit tests against the drop-in
# package on a GPU box.  The test files are copied from /root/reference into a
# scratch directory (git-ignored, deleted afterwards), the import name `linkcert`
# is bound to paper_2106_12655_b200 by tools/refshim, and the log is kept.
#   bash tools/run_reference_tests.sh profiles/r02/reference_tests.log
set -e
LOG=${1:-profiles/r02/reference_tests.log}
rm -rf _reftests && mkdir -p _reftests
# default: the hot-path files SURVEY §8(c) names first; REFTESTS="..." to choose (e.g. the
# data-model / digest / acceptance / BH files)
REFTESTS=${REFTESTS:-"test_direct.py test_kernels.py test_certify.py test_pls.py test_discretize.py"}
for f in conftest.py $REFTESTS; do
  cp /root/reference/pkg/tests/$f _reftests/
done
/usr/local/graft/bin/gpurun --timeout 900 -- "cd _reftests && PYTHONPATH=../tools/refshim:.. python -m pytest -p no:cacheprovider -p ref_plugin -q -rf . > ../gpurun_out/reference_tests.log 2>&1; echo rc=\$?" || true
rm -rf _reftests
cp gpurun_out/reference_tests.log "$LOG"
tail -30 "$LOG"
