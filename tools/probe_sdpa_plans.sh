# cuDNN SDPA plan timings at the 8B shape (CFT_VERBOSE prints every candidate during autotune)
CFT_VERBOSE=1 timeout 600 python -c "
import sys; sys.path.insert(0, '.')
from paper_2605_21177_b200.engine import ChunkEngine, LlamaModel, TrainOptions
from paper_2605_21177_b200.plan import ScheduleConfig
m = LlamaModel.llama3_8b(layers=1)
e = ChunkEngine(m, None, 8, TrainOptions(schedule=ScheduleConfig(K=4, T=1, total_steps=1), dtype='bf16'), seed=1)
" 2>&1 | grep -i "sdpa" | head -40
