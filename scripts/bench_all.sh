# Round bench lines: every config on one GPU (default bench + per-config lines)
# usage: bash scripts/bench_all.sh TAG
set -e
TAG=${1:-rx}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_${TAG}_17_6.json 2> gpurun_out/bench_${TAG}_17_6.err
python bench.py --config 13_4 > gpurun_out/bench_${TAG}_13_4.json 2> gpurun_out/bench_${TAG}_13_4.err
python bench.py --config 21_8 --steps 3 > gpurun_out/bench_${TAG}_21_8.json 2> gpurun_out/bench_${TAG}_21_8.err
python bench.py --config 23_9 --steps 3 > gpurun_out/bench_${TAG}_23_9.json 2> gpurun_out/bench_${TAG}_23_9.err
tail -c 400 gpurun_out/bench_${TAG}_*.json
