# One verification call: build, smoke, full GPU suite, default bench line.
# tools/gpu_round.sh <tag>   (outputs gpurun_out/<tag>_*)
cd $GRAFT_REPO_ROOT
tag=${1:-round}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/${tag}_tests.log 2>&1
tail -3 gpurun_out/${tag}_tests.log
