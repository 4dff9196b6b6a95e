import sys; sys.path.insert(0, ".")
from paper_2506_07639_b200.engine import Engine
e = Engine("7b", dtype="bf16", kv_pages=64, vision=True)
for i in range(2): e.vision_encode(i)
