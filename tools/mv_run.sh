# Build single-module variants, pack them, and time them on the GPU box (tools/modvar.py):
#   bash tools/mv_run.sh TAG OUT.jsonl "TIME_ARGS" NAME=KNOBS ...
set -e -o pipefail
TAG=$1; OUTJ=$2; TARGS=$3; shift 3
export MODVAR_DIR=/tmp/modvar_run
rm -rf $MODVAR_DIR/$TAG
python tools/modvar.py build $TAG "$@" 2>&1 | grep -E "^[A-Za-z0-9_]+$|  const |  mat |  ws |rror" | grep -v "^Remark"
ls $MODVAR_DIR/$TAG/*.so > /dev/null
rm -f $MODVAR_DIR/$TAG/*.o build_modvar.tgz
(cd $MODVAR_DIR && tar czf /root/repo/build_modvar.tgz --transform 's,^,build_modvar/,' $TAG)
/usr/local/graft/bin/gpurun --timeout 1500 -- "tar xzf build_modvar.tgz && python tools/modvar.py time $TAG $OUTJ $TARGS 2>&1 | grep ' ms '" 2>&1 | grep -E " ms |status=|rror"
rm -f build_modvar.tgz
