timeout 900 python tools/win_fit.py 4 > gpurun_out/win_fit.jsonl 2> gpurun_out/win_fit.err
echo fit=$?
