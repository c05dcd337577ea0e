python bench.py > gpurun_out/default.json 2> gpurun_out/default.err; echo "ours rc=$?"
python bench.py --impl reference > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
cat gpurun_out/default.json; echo; cat gpurun_out/ref.json
