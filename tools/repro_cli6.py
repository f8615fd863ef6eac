import random, string, sys
sys.path.insert(0, '.')
from paper_1407_6603_b200.pipeline import sort_text
ALNUM = (string.ascii_letters + string.digits).encode()
rng = random.Random(66)
words = [bytes(rng.choices(ALNUM, k=rng.randint(1, 40))) for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 48000)]
text = b" ".join(words)
out = sort_text(text)
exp = b"".join(w + b"\n" for w in sorted(words, key=lambda w: (len(w), w)))
print("ok" if out == exp else "MISMATCH", len(text))
