set -x
timeout 900 python tools/parity_report.py > gpurun_out/parity.jsonl 2> gpurun_out/parity.err
echo done
