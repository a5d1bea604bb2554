for rep in 1 2 3; do
python tools/probe_cg.py --n 256 --iters 300 --repeat 2
python tools/probe_cg.py --n 512 --iters 60 --repeat 2
python tools/probe_cg.py --n 128 --iters 300 --repeat 2
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
