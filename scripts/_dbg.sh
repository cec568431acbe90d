timeout 120 python scripts/timeline.py; SAP_SIDE_STREAM=1 timeout 120 python scripts/timeline.py
