set -x
python tools/ubench_conv.py 0: 1: 2: 3:
python tools/acct_conv.py
python tools/cta_timeline.py
