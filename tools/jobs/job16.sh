timeout 200 python tools/mb_order.py
