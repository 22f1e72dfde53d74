# Run the reference's own tests (/root/reference/pkg/tests) against this
# package.  Stage (here, where /root/reference exists):  bash scripts/run_ref_suite.sh stage
# Run (GPU box; the staged copy travels in build/):      bash scripts/run_ref_suite.sh run
set -e
case "$1" in
  stage)
    rm -rf build/ref_suite && mkdir -p build/ref_suite
    cp /root/reference/pkg/tests/*.py build/ref_suite/
    ;;
  run)
    mkdir -p gpurun_out
    PYTHONPATH=scripts:$PYTHONPATH python -m pytest -p splinemat_alias build/ref_suite -q -rfEs \
        -p no:cacheprovider --rootdir build/ref_suite > gpurun_out/ref_suite.log 2>&1 || true
    tail -60 gpurun_out/ref_suite.log
    ;;
esac
