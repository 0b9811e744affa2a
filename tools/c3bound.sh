export CFG=3 WT=256
python tools/v7env.py
ENVS="NSDGT_DBG=128" python tools/v7env.py
ENVS="NSDGT_DBG=128" bash tools/altrun.sh tools/libnsdgt_xp_NORING.so tools/v7env.py
bash tools/altrun.sh tools/libnsdgt_xp_NORING.so tools/v7env.py
