"""Float64 numpy oracle of the MetaTune cost-model hot path (TEST INFRASTRUCTURE).

A restatement of the reference algorithm, kept deliberately independent of
the product package (its own knob tables, encoder and model math) so that it
checks the product's host logic as well as the device kernels.  Citations are
to /root/reference/pkg/src/kerntune/<file>:<line>.

Model parameters are a plain dict:
    {"gcn": [W (d_in, d_out), ...], "agg": (d,), "head_w": [W, ...],
     "head_b": [b, ...], "fmean": (F,), "fstd": (F,), "lmean": float, "lstd": float}
"""

from __future__ import annotations

import math

import numpy as np

F = 12
AXES = {
    "conv1d": ("x", "f", "rc", "rx"),
    "transpose1d": ("x", "f", "rc", "rx"),
    "conv2d": ("x", "y", "f", "rc", "rx", "ry"),
    "transpose2d": ("x", "y", "f", "rc", "rx", "ry"),
    "winograd": ("x", "y", "f", "rc", "rx", "ry"),
    "depthwise": ("x", "y", "f", "rx", "ry"),
}
CANON = ("x", "y", "f", "rc", "rx", "ry")
REDUCE = ("rc", "rx", "ry")
CARD = {"x": 140, "y": 140, "f": 120, "rc": 8, "rx": 2, "ry": 2}


# --- knob space (kernels.py:168-286) --------------------------------------------


def extents(op, input_size, in_ch, out_ch, ksize, stride=3, padding=1) -> dict:
    """kernels.py:160-187."""
    conv = max((input_size + 2 * padding - ksize) // stride + 1, 1)
    tr = max((input_size - 1) * stride - 2 * padding + ksize, 1)
    if op in ("conv1d", "conv2d", "depthwise"):
        s = conv
    elif op in ("transpose1d", "transpose2d"):
        s = tr
    else:
        s = max(math.ceil(conv / 2), 1)
    e = {"x": s, "y": s, "f": out_ch}
    if op == "winograd":
        e.update(rc=in_ch, rx=4, ry=4)
    elif op == "depthwise":
        e.update(rx=ksize, ry=ksize)
    else:
        e.update(rc=in_ch, rx=ksize, ry=ksize)
    return {a: e[a] for a in AXES[op]}


def tile_list(extent: int, count: int) -> list:
    """kernels.py:190-228: divisors, spread-thinned or padded past extent."""
    divs = [d for d in range(1, extent + 1) if extent % d == 0]
    if len(divs) < count:
        return divs + [extent + i + 1 for i in range(count - len(divs))]
    if count == 1:
        return [divs[0]]
    pick, used = [], set()
    for i in range(count):
        j = round(i * (len(divs) - 1) / (count - 1))
        while j in used:
            j += 1
        used.add(j)
        pick.append(divs[j])
    return pick


def knob_lists(op, ext: dict) -> list:
    """kernels.py:231-260 (uncapped): [(name, values)] in knob order."""
    out = [(f"tile_{a}", tile_list(ext[a], CARD[a])) for a in AXES[op]]
    out.append(("auto_unroll_max_step", [0, 512, 1500]))
    out.append(("unroll_explicit", [0, 1]))
    return out


def decode(cards, idx) -> np.ndarray:
    """kernels.py:278-286 vectorised: index -> (B, n_knobs) choices."""
    idx = np.asarray(idx, dtype=np.int64).copy()
    out = np.zeros((idx.shape[0], len(cards)), dtype=np.int64)
    for j in range(len(cards) - 1, -1, -1):
        out[:, j] = idx % cards[j]
        idx //= cards[j]
    return out


# --- encoder (graphs.py:89-126, 305-351) ------------------------------------------


def context_features(e, lvl, red, unr, strd) -> np.ndarray:
    n = e.shape[-1]
    touched = np.ones_like(e)
    if n > 1:
        rev = np.cumprod(e[..., ::-1], axis=-1)[..., ::-1]
        touched[..., :-1] = rev[..., 1:]
    arith = 2.0 * touched
    lg = lambda v: np.log2(np.maximum(v, 1.0))
    depth = np.broadcast_to(np.arange(1, n + 1, dtype=np.float64), e.shape)
    pos = np.broadcast_to(np.arange(n, dtype=np.float64) / max(n - 1, 1), e.shape)
    cols = [e, lg(e), lvl, red, unr, strd, touched, lg(touched), arith, lg(arith), depth, pos]
    return np.stack(np.broadcast_arrays(*cols), axis=-1)


def loop_features(op, ext, knobs, choices) -> np.ndarray:
    """(B, n_loops, 12) raw features; loops = outer axes then inner axes."""
    b = choices.shape[0]
    axes = AXES[op]
    na = len(axes)
    vals = {name: np.asarray(v, dtype=np.int64)[choices[:, j]] for j, (name, v) in enumerate(knobs)}
    e = np.empty((b, 2 * na))
    lvl = np.zeros((b, 2 * na))
    red = np.zeros((b, 2 * na))
    unr = np.zeros((b, 2 * na))
    strd = np.ones((b, 2 * na))
    auto = vals["auto_unroll_max_step"]
    expl = vals["unroll_explicit"].astype(bool)
    for k, a in enumerate(axes):
        t = np.clip(vals[f"tile_{a}"], 1, ext[a])
        e[:, k] = -(-ext[a] // t)
        e[:, na + k] = t
        lvl[:, na + k] = 1.0
        if a in REDUCE:
            red[:, k] = red[:, na + k] = 1.0
        unr[:, na + k] = (expl & (auto > 0) & (t <= auto)).astype(np.float64)
        strd[:, k] = t
    return context_features(e, lvl, red, unr, strd)


def layout(op, super_graph: bool):
    """graphs.py:278-302: (adjacency fp64, iterval rows, mask) for raw or super."""
    def names(axes):
        return [f"{a}_{s}" for s in ("outer", "inner") for a in CANON if a in axes]

    loop_names = names(set(AXES[op]))
    if super_graph:
        slots = names(set(CANON))
        rows = np.array([2 + 2 * slots.index(nm) for nm in loop_names])
        n_pairs = len(slots)
    else:
        rows = np.array([2 + 2 * i for i in range(len(loop_names))])
        n_pairs = len(loop_names)
    n = 1 + 2 * n_pairs
    edges = [(0, 1 + 2 * i) for i in range(n_pairs)] + [(1 + 2 * i, 2 + 2 * i) for i in range(n_pairs)]
    adj = normalized_adjacency(n, edges)
    mask = np.zeros(n, dtype=bool)
    mask[rows] = True
    return adj, rows, mask


def normalized_adjacency(n, edges) -> np.ndarray:
    """graphs.py:234-241."""
    a = np.zeros((n, n))
    for s, d in edges:
        a[s, d] = 1.0
        a[d, s] = 1.0
    np.fill_diagonal(a, a.diagonal() + 1.0)
    dinv = 1.0 / np.sqrt(a.sum(axis=1))
    return a * dinv[:, None] * dinv[None, :]


def encode(op, ext, knobs, choices, n_nodes, rows) -> np.ndarray:
    """encode_batch (graphs.py:305-351): (B, N, 12) fp64, zeros off the iterval rows."""
    feats = loop_features(op, ext, knobs, choices)
    out = np.zeros((choices.shape[0], n_nodes, F))
    out[:, rows, :] = feats
    return out


# --- model forward (model.py:108-203) ------------------------------------------------


def init_params(rng, feature_dim=F, gcn_dims=(32, 32), head_hidden=(64, 64)) -> dict:
    """model.py:71-96, same draw order: gcn weights, then (w_i, b_i) pairs."""
    def u(fan_in, shape):
        s = 1.0 / math.sqrt(fan_in)
        return rng.uniform(-s, s, size=shape)

    dims = (feature_dim,) + tuple(gcn_dims)
    gcn = [u(dims[i], (dims[i], dims[i + 1])) for i in range(len(dims) - 1)]
    hd = (2 * dims[-1],) + tuple(head_hidden) + (1,)
    hw, hb = [], []
    for i in range(len(hd) - 1):
        hw.append(u(hd[i], (hd[i], hd[i + 1])))
        hb.append(u(hd[i], (hd[i + 1],)))
    return {"gcn": gcn, "agg": np.ones(dims[-1]), "head_w": hw, "head_b": hb,
            "fmean": np.zeros(feature_dim), "fstd": np.ones(feature_dim),
            "lmean": 0.0, "lstd": 1.0}


def normalize(p, x, mask) -> np.ndarray:
    out = np.zeros_like(x)
    out[..., mask, :] = (x[..., mask, :] - p["fmean"]) / p["fstd"]
    return out


def embed_batch(p, feats, mask, adj) -> np.ndarray:
    """model.py:185-194."""
    h = normalize(p, feats, mask)
    for w in p["gcn"]:
        h = np.maximum(np.einsum("nm,bmf,fd->bnd", adj, h, w, optimize=True), 0.0)
    return np.concatenate([(h * p["agg"]).sum(axis=1), h.max(axis=1)], axis=1)


def gcn_forward_batch(p, feats, mask, adj) -> np.ndarray:
    """gcn_forward (model.py:127-133) over a batch sharing one adjacency: H_L (B, N, d_L)."""
    h = normalize(p, feats, mask)
    for w in p["gcn"]:
        h = np.maximum(np.einsum("nm,bmf,fd->bnd", adj, h, w, optimize=True), 0.0)
    return h


def aggregate_batch(h, agg) -> np.ndarray:
    """aggregate (model.py:136-141) per graph: [sum_n a * h_n, max_n h_n]."""
    return np.concatenate([(h * agg).sum(axis=1), h.max(axis=1)], axis=1)


def head_forward_batch(u, hw, hb) -> np.ndarray:
    """model.py:197-203."""
    a = u
    for i, (w, b) in enumerate(zip(hw, hb)):
        z = a @ w + b
        a = z if i == len(hw) - 1 else np.maximum(z, 0.0)
    return a[:, 0]


def score(p, feats, mask, adj) -> np.ndarray:
    return head_forward_batch(embed_batch(p, feats, mask, adj), p["head_w"], p["head_b"])


def normalize_label(p, gflops) -> float:
    """model.py:99-101 with LABEL_FLOOR 1e-3 (model.py:23)."""
    return (math.log2(max(gflops, 1e-3)) - p["lmean"]) / p["lstd"]


# --- gradients (model.py:218-285) ------------------------------------------------------


def grad(p, graphs, labels, scope="all"):
    """(loss, grads dict) of batch MSE over graphs = [(X raw, adj, mask)]."""
    g = {"gcn": [np.zeros_like(w) for w in p["gcn"]], "agg": np.zeros_like(p["agg"]),
         "head_w": [np.zeros_like(w) for w in p["head_w"]],
         "head_b": [np.zeros_like(b) for b in p["head_b"]]}
    total, inv_b = 0.0, 1.0 / len(graphs)
    last = len(p["head_w"]) - 1
    for (x_raw, adj, mask), label in zip(graphs, labels):
        x = normalize(p, x_raw, mask)
        hs, zs, h = [x], [], x
        for w in p["gcn"]:
            z = adj @ h @ w
            h = np.maximum(z, 0.0)
            zs.append(z)
            hs.append(h)
        u = np.concatenate([(h * p["agg"]).sum(axis=0), h.max(axis=0)])
        a, acts, zh = u, [u], []
        for i, (w, b) in enumerate(zip(p["head_w"], p["head_b"])):
            z = a @ w + b
            a = z if i == last else np.maximum(z, 0.0)
            zh.append(z)
            acts.append(a)
        pred = float(a[0])
        y = normalize_label(p, label)
        total += (pred - y) ** 2
        da = np.array([2.0 * (pred - y) * inv_b])
        for i in range(last, -1, -1):
            dz = da if i == last else da * (zh[i] > 0.0)
            g["head_w"][i] += np.outer(acts[i], dz)
            g["head_b"][i] += dz
            da = dz @ p["head_w"][i].T
        if scope == "head_only":
            continue
        d = p["agg"].shape[0]
        ds, dmx = da[:d], da[d:]
        g["agg"] += hs[-1].sum(axis=0) * ds
        dh = np.tile(p["agg"] * ds, (hs[-1].shape[0], 1))
        dh[np.argmax(hs[-1], axis=0), np.arange(d)] += dmx  # first-index argmax (model.py:276)
        for li in range(len(p["gcn"]) - 1, -1, -1):
            dz = dh * (zs[li] > 0.0)
            g["gcn"][li] += (adj @ hs[li]).T @ dz
            dh = adj @ (dz @ p["gcn"][li].T)
    return total * inv_b, g


def sgd(p, g, lr) -> dict:
    """model.py:288-310 on the full state."""
    out = dict(p)
    out["gcn"] = [w - lr * d for w, d in zip(p["gcn"], g["gcn"])]
    out["agg"] = p["agg"] - lr * g["agg"]
    out["head_w"] = [w - lr * d for w, d in zip(p["head_w"], g["head_w"])]
    out["head_b"] = [b - lr * d for b, d in zip(p["head_b"], g["head_b"])]
    return out


# --- flat head engine (model.py:328-432) -------------------------------------------------


def head_to_vec(hw, hb) -> np.ndarray:
    return np.concatenate([np.concatenate([w.ravel(), b]) for w, b in zip(hw, hb)])


def vec_to_head(vec, shapes):
    """shapes = [(d_in, d_out), ...]; returns (weights, biases) views."""
    ws, bs, off = [], [], 0
    for din, dout in shapes:
        ws.append(vec[off : off + din * dout].reshape(din, dout))
        off += din * dout
        bs.append(vec[off : off + dout])
        off += dout
    assert off == vec.size, "flat head vector has the wrong length"
    return ws, bs


def head_loss_grad(vec, shapes, u, y):
    """model.py:358-389: (mse, d mse / d vec)."""
    ws, bs = vec_to_head(vec, shapes)
    last = len(ws) - 1
    acts, signs, a = [u], [], u
    for i, (w, b) in enumerate(zip(ws, bs)):
        z = a @ w + b
        if i == last:
            a = z
        else:
            signs.append(z > 0.0)
            a = np.maximum(z, 0.0)
        acts.append(a)
    resid = acts[-1][:, 0] - y
    n = y.shape[0]
    mse = float(resid @ resid / n)
    da = (2.0 / n) * resid[:, None]
    parts = [None] * len(ws)
    for i in range(last, -1, -1):
        dz = da if i == last else da * signs[i]
        parts[i] = np.concatenate([(acts[i].T @ dz).ravel(), dz.sum(axis=0)])
        da = dz @ ws[i].T
    return mse, np.concatenate(parts)


def head_hvp(vec, shapes, u, y, v) -> np.ndarray:
    """model.py:392-432: forward-over-reverse H v, ReLU masks constant."""
    ws, bs = vec_to_head(vec, shapes)
    vw, vb = vec_to_head(v, shapes)
    last = len(ws) - 1
    acts, tacts, signs = [u], [np.zeros_like(u)], []
    a, ta = u, np.zeros_like(u)
    for i, (w, b) in enumerate(zip(ws, bs)):
        z = a @ w + b
        tz = ta @ w + a @ vw[i] + vb[i]
        if i == last:
            a, ta = z, tz
        else:
            s = z > 0.0
            signs.append(s)
            a, ta = np.maximum(z, 0.0), tz * s
        acts.append(a)
        tacts.append(ta)
    n = y.shape[0]
    da = (2.0 / n) * (acts[-1][:, 0] - y)[:, None]
    tda = (2.0 / n) * tacts[-1][:, 0][:, None]
    parts = [None] * len(ws)
    for i in range(last, -1, -1):
        dz = da if i == last else da * signs[i]
        tdz = tda if i == last else tda * signs[i]
        gw = tacts[i].T @ dz + acts[i].T @ tdz
        parts[i] = np.concatenate([gw.ravel(), tdz.sum(axis=0)])
        da = dz @ ws[i].T
        tda = tdz @ ws[i].T + dz @ vw[i].T
    return np.concatenate(parts)


# --- meta-learning (meta.py:81-297) ------------------------------------------------------


def dataset_norms(feature_rows, labels_gflops):
    """meta.py:81-101 from stacked iterval rows (R, 12) and raw GFLOPS labels."""
    mean = feature_rows.mean(axis=0)
    std = feature_rows.std(axis=0)
    std = np.where(std < 1e-12, 1.0, std)
    logs = [math.log2(max(v, 1e-3)) for v in labels_gflops]
    lm, ls = float(np.mean(logs)), float(np.std(logs))
    return mean, std, lm, (ls if ls >= 1e-12 else 1.0)


def maml_outer_grad(theta, sgrad, qgrad, alpha, inner_steps, first_order, shvp=None):
    """meta.py:167-196."""
    thetas, ls0 = [theta], None
    for _ in range(inner_steps):
        ls, gs = sgrad(thetas[-1])
        if ls0 is None:
            ls0 = ls
        thetas.append(thetas[-1] - alpha * gs)
    lq, v = qgrad(thetas[-1])
    if not first_order:
        for k in range(inner_steps - 1, -1, -1):
            v = v - alpha * shvp(thetas[k], v)
    return ls0, lq, v, thetas[-1]


def meta_step_embedded(theta, shapes, tasks, alpha, beta, inner_steps=1, first_order=True):
    """meta.py:223-257 on pre-embedded tasks [(us, ys, uq, yq)]: theta - beta * sum_i g_i."""
    outer = np.zeros_like(theta)
    sl, ql = [], []
    for us, ys, uq, yq in tasks:
        ls, lq, g, _ = maml_outer_grad(
            theta,
            lambda t: head_loss_grad(t, shapes, us, ys),
            lambda t: head_loss_grad(t, shapes, uq, yq),
            alpha, inner_steps, first_order,
            lambda t, v: head_hvp(t, shapes, us, ys, v),
        )
        outer += g
        sl.append(ls)
        ql.append(lq)
    return theta - beta * outer, float(np.mean(sl)), float(np.mean(ql))


def fine_tune_embedded(theta, shapes, u, y, alpha, steps):
    """meta.py:274-282."""
    for _ in range(steps):
        _, g = head_loss_grad(theta, shapes, u, y)
        theta = theta - alpha * g
    return theta


def sample_task_indices(class_members: dict, n_way, k_shot, meta_batch, rng):
    """meta.py:136-161 on index lists: eligible classes sorted; choice then per-class
    permutation, in the reference's draw order.  Returns [(support idx, query idx)]."""
    eligible = sorted(c for c, m in class_members.items() if len(m) >= k_shot + 1)
    tasks = []
    for _ in range(meta_batch):
        classes = [eligible[int(i)] for i in rng.choice(len(eligible), n_way, replace=False)]
        sup, qry = [], []
        for c in classes:
            pool = class_members[c]
            perm = rng.permutation(len(pool))
            sup += [pool[int(i)] for i in perm[:k_shot]]
            q = min(k_shot, len(pool) - k_shot)
            qry += [pool[int(i)] for i in perm[k_shot : k_shot + q]]
        tasks.append((sup, qry))
    return tasks


# --- ranking (search.py:257-264) ------------------------------------------------------------


def rank_history(indices, scores, visited, count) -> list:
    ranked = sorted(((int(i), float(e)) for i, e in zip(indices, scores) if int(i) not in visited),
                    key=lambda t: (-t[1], t[0]))
    return [i for i, _ in ranked[:count]]


# --- simulated-annealing exploration (search.py:177-281) ------------------------------------


def space_multipliers(cards) -> np.ndarray:
    """_space_multipliers (search.py:177-182): knob 0 most significant."""
    mult = np.ones(len(cards), dtype=np.int64)
    for j in range(len(cards) - 2, -1, -1):
        mult[j] = mult[j + 1] * cards[j + 1]
    return mult


def draw_unvisited(size: int, visited: set, count: int, rng) -> list:
    """draw_unvisited (search.py:185-211): distinct unvisited indices, same RNG draws."""
    remaining = size - len(visited)
    count = min(count, max(remaining, 0))
    if count <= 0:
        return []
    if size <= 65536:
        unvisited = np.array([i for i in range(size) if i not in visited], dtype=np.int64)
        pick = rng.choice(len(unvisited), size=count, replace=False)
        return [int(unvisited[i]) for i in pick]
    out, chosen = [], set()
    while len(out) < count:
        need = count - len(out)
        for v in rng.integers(0, size, size=need + 8):
            i = int(v)
            if i not in visited and i not in chosen:
                chosen.add(i)
                out.append(i)
                if len(out) == count:
                    break
    return out


def sa_draws(rng, cards, n_chains, steps):
    """The per-step random draws of sa_explore (search.py:233-237), in the reference's order."""
    cards = np.asarray(cards, dtype=np.int64)
    out = []
    for _ in range(steps):
        knob = rng.integers(0, len(cards), size=n_chains)
        nudge = rng.random(n_chains) < 0.5
        delta = rng.integers(0, 2, size=n_chains) * 2 - 1
        resample = rng.integers(0, cards[knob])
        u = rng.random(n_chains)
        out.append((knob, nudge, delta, resample, u))
    return out


def sa_explore(predict_idx, cards, size, sched, visited, rng) -> dict:
    """sa_explore (search.py:202-254); predict_idx maps int64 config indices -> float64 scores.
    sched = (initial_temp, cooling, steps_per_round, parallel_chains)."""
    t0, cooling, steps, chains = sched
    starts = draw_unvisited(size, visited, chains, rng)
    if not starts:
        return {}
    cards = np.asarray(cards, dtype=np.int64)
    mult = space_multipliers(cards)
    cur = decode(cards, np.array(starts, dtype=np.int64))
    n = cur.shape[0]
    energy = np.asarray(predict_idx((cur * mult).sum(axis=1)), dtype=np.float64)
    history = {int(i): float(e) for i, e in zip((cur * mult).sum(axis=1), energy)}
    temp = t0
    rows = np.arange(n)
    for knob, nudge, delta, resample, u in sa_draws(rng, cards, n, steps):
        nxt = cur.copy()
        stepped = np.clip(cur[rows, knob] + delta, 0, cards[knob] - 1)
        nxt[rows, knob] = np.where(nudge, stepped, resample)
        idx = (nxt * mult).sum(axis=1)
        e_new = np.asarray(predict_idx(idx), dtype=np.float64)
        for i, e in zip(idx, e_new):
            history[int(i)] = float(e)
        downhill_p = np.exp(np.minimum((e_new - energy) / temp, 0.0))
        accept = (e_new >= energy) | (u < downhill_p)
        cur = np.where(accept[:, None], nxt, cur)
        energy = np.where(accept, e_new, energy)
        temp = max(temp * cooling, 1e-9)
    return history


def sa_propose(predict_idx, cards, size, sched, visited, rng, batch) -> list:
    """sa_propose (search.py:266-281): explore, rank, top up with unvisited draws."""
    history = sa_explore(predict_idx, cards, size, sched, visited, rng)
    picks = rank_history(np.array(list(history.keys()), dtype=np.int64),
                         np.array(list(history.values())), visited, batch)
    if len(picks) < batch:
        picks += draw_unvisited(size, visited | set(picks), batch - len(picks), rng)
    return picks


# --- GP surrogate + batch UCB (search.py:39-159, 284-340) ------------------------------------

GP_LENGTHSCALES = (0.1, 0.3, 1.0, 3.0)  # search.py:37
GP_MAX_JITTER = 1e-1                     # search.py:38


def gp_kernel(x1, x2, ls) -> np.ndarray:
    """RBF on lengthscale-scaled coordinates (search.py:72-76)."""
    a = x1 / ls
    b = x2 / ls
    d2 = (a * a).sum(axis=1)[:, None] + (b * b).sum(axis=1)[None, :] - 2.0 * a @ b.T
    return np.exp(-0.5 * np.maximum(d2, 0.0))


def gp_chol(k, noise):
    """Cholesky of k + nv I with tenfold jitter escalation (search.py:79-91); None when
    even MAX_JITTER fails (the reference raises NumericError)."""
    nv = noise
    while True:
        try:
            return np.linalg.cholesky(k + nv * np.eye(k.shape[0])), nv
        except np.linalg.LinAlgError:
            pass
        if nv >= GP_MAX_JITTER:
            return None, nv
        nv *= 10.0


def gp_fit(x, y, noise, ls=None):
    """(lengthscales, L, alpha, noise) maximising the marginal likelihood over the grid
    (search.py:94-121); ls fixes the lengthscales instead."""
    n, d = x.shape
    cands = [np.full(d, v) for v in GP_LENGTHSCALES] if ls is None else [np.asarray(ls, dtype=np.float64)]
    best = None
    for c in cands:
        l, nv = gp_chol(gp_kernel(x, x, c), noise)
        z = np.linalg.solve(l, y)  # cho_solve: L z = y, L^T alpha = z
        alpha = np.linalg.solve(l.T, z)
        mll = -0.5 * float(y @ alpha) - float(np.log(np.diag(l)).sum()) - 0.5 * n * math.log(2.0 * math.pi)
        if best is None or mll > best[0]:
            best = (mll, c, l, alpha, nv)
    return best[1], best[2], best[3], best[4]


def gp_posterior(x, ls, l, alpha, xp):
    """(mean, var, cov) of the latent function at xp (search.py:129-157)."""
    kxn = gp_kernel(x, xp, ls)
    v = np.linalg.solve(l, kxn)
    mean = kxn.T @ alpha
    var = np.maximum(1.0 - (v * v).sum(axis=0), 0.0)
    cov = gp_kernel(xp, xp, ls) - v.T @ v
    return mean, var, cov


def ucb_batch(mean, cov, noise, beta, take) -> list:
    """Sequential UCB with hallucinated downdates (search.py:324-340): positions into
    the (sorted) pool, in pick order."""
    var = np.maximum(np.diag(cov).copy(), 0.0)
    cov = cov.copy()
    active = np.ones(len(mean), dtype=bool)
    out = []
    for _ in range(take):
        ucb = mean + math.sqrt(beta) * np.sqrt(np.maximum(var, 0.0))
        ucb[~active] = -np.inf
        z = int(np.argmax(ucb))
        out.append(z)
        active[z] = False
        denom = var[z] + noise
        if denom > 0.0:
            c = cov[:, z].copy()
            var = np.maximum(var - c * c / denom, 0.0)
            cov = cov - np.outer(c, c) / denom
    return out
