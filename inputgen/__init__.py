"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it draws random action
tensors with numpy and builds canonical state records (SURVEY §8b layout) from
ASCII maps for fixtures.  Both the oracle (``oracle/``) and the product
(``paper_2407_19396_b200``) consume what it produces; neither is imported here.

Canonical per-env record:
  H*W cells as (type, colour, state) in MiniGrid's encoding, row-major
  (y outer, x inner); agent x, y, dir; carry (type, colour), (1, 0) = nothing;
  step_count u16 LE; episode u32 LE; prev_done u8; DynObs: n x (x, y).
"""
from __future__ import annotations

import numpy as np

# MiniGrid OBJECT_TO_IDX / COLOR_TO_IDX / STATE_TO_IDX values (data format).
EMPTY, WALL, FLOOR, DOOR, KEY, BALL, BOX, GOAL, LAVA = 1, 2, 3, 4, 5, 6, 7, 8, 9
RED, GREEN, BLUE, PURPLE, YELLOW, GREY = 0, 1, 2, 3, 4, 5
OPEN, CLOSED, LOCKED = 0, 1, 2

# ASCII legend for fixture maps.  Door/key/ball colours come from `colors`.
_LEGEND = {
    "#": (WALL, GREY, 0),
    ".": (EMPTY, 0, 0),
    "A": (EMPTY, 0, 0),  # agent cell (nothing under it)
    "G": (GOAL, GREEN, 0),
    "V": (LAVA, RED, 0),
    "K": (KEY, YELLOW, 0),
    "B": (BALL, BLUE, 0),
    "O": (DOOR, YELLOW, OPEN),
    "D": (DOOR, YELLOW, CLOSED),
    "L": (DOOR, YELLOW, LOCKED),
}


def random_actions(seed: int, steps: int, n: int, n_actions: int, high: int | None = None) -> np.ndarray:
    """uint8[steps, n] uniform over [0, high or n_actions) from numpy's PCG64."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, high if high is not None else n_actions, size=(steps, n), dtype=np.uint8)


def record_from_map(rows: list[str], agent_dir: int, *, carry=(EMPTY, 0), step_count: int = 0,
                    episode: int = 0, prev_done: int = 0, colors: dict | None = None,
                    balls: list[tuple[int, int]] | None = None,
                    target: tuple[int, int] | None = None) -> np.ndarray:
    """Canonical record for one env from an ASCII map (rows = y, columns = x);
    `target` = GoToDoor's target door (x, y), appended last."""
    H, W = len(rows), len(rows[0])
    colors = colors or {}
    out = []
    ax = ay = None
    for y, row in enumerate(rows):
        assert len(row) == W
        for x, ch in enumerate(row):
            t, c, s = _LEGEND[ch]
            if ch in colors:
                c = colors[ch]
            if ch == "A":
                ax, ay = x, y
            out += [t, c, s]
    assert ax is not None, "map needs an 'A'"
    out += [ax, ay, agent_dir, carry[0], carry[1]]
    out += list(int(step_count).to_bytes(2, "little"))
    out += list(int(episode).to_bytes(4, "little"))
    out += [prev_done]
    for bx, by in balls or []:
        out += [bx, by]
    if target is not None:
        out += list(target)
    return np.array(out, np.uint8)


def decode_record(rec: np.ndarray, H: int, W: int, n_obstacles: int = 0) -> dict:
    """Split a canonical record into named fields (inverse of record_from_map)."""
    rec = np.asarray(rec, np.uint8)
    cells = rec[: 3 * H * W].reshape(H, W, 3)
    p = 3 * H * W
    d = {
        "cells": cells,
        "agent": (int(rec[p]), int(rec[p + 1]), int(rec[p + 2])),
        "carry": (int(rec[p + 3]), int(rec[p + 4])),
        "step_count": int(rec[p + 5]) | (int(rec[p + 6]) << 8),
        "episode": int.from_bytes(bytes(rec[p + 7: p + 11]), "little"),
        "prev_done": int(rec[p + 11]),
    }
    q = p + 12
    d["balls"] = [(int(rec[q + 2 * i]), int(rec[q + 2 * i + 1])) for i in range(n_obstacles)]
    return d


def random_records(seed: int, n: int, H: int, W: int, max_steps: int, n_obstacles: int = 0,
                   p_prev_done: float = 0.0, open_edge: bool = False) -> np.ndarray:
    """n canonical records of random but legal states: wall border, random
    interior objects (walls, doors in all three states, keys, balls, boxes,
    goals, lava, floor), the agent on a walkable interior cell, a random
    carried object, random step count.  With n_obstacles > 0 (DynObs) exactly
    that many blue balls are listed (extra balls may still appear as static
    objects).  open_edge (GoToDoor records): the border cells are random too,
    the agent may stand on any walkable cell, and a random target door
    position (x, y) inside the grid ends the record."""
    rng = np.random.default_rng(seed)
    kinds = np.array([EMPTY, WALL, DOOR, KEY, BALL, BOX, GOAL, LAVA, FLOOR])
    probs = np.array([0.42, 0.16, 0.12, 0.07, 0.06, 0.04, 0.05, 0.05, 0.03])
    per = 3 * H * W + 12 + 2 * n_obstacles + (2 if open_edge else 0)
    out = np.zeros((n, per), np.uint8)
    m = 0 if open_edge else 1
    for e in range(n):
        cells = np.zeros((H, W, 3), np.uint8)
        cells[:, :, 0] = WALL
        cells[:, :, 1] = GREY
        for y in range(m, H - m):
            for x in range(m, W - m):
                k = rng.choice(kinds, p=probs)
                c = int(rng.integers(0, 6))
                if k == EMPTY:
                    cells[y, x] = (EMPTY, 0, 0)
                elif k == DOOR:
                    cells[y, x] = (DOOR, c, int(rng.integers(0, 3)))
                else:
                    cells[y, x] = (k, c, 0)
        walk = [(x, y) for y in range(m, H - m) for x in range(m, W - m)
                if cells[y, x, 0] in (EMPTY, FLOOR, GOAL, LAVA) or (cells[y, x, 0] == DOOR and cells[y, x, 2] == OPEN)]
        if not walk:
            x, y = 1, 1
            cells[y, x] = (EMPTY, 0, 0)
            walk = [(1, 1)]
        ax, ay = walk[int(rng.integers(len(walk)))]
        balls = []
        if n_obstacles:
            free = [(x, y) for y in range(1, H - 1) for x in range(1, W - 1) if (x, y) != (ax, ay)]
            pick = rng.permutation(len(free))[:n_obstacles]
            for i in pick:
                bx, by = free[i]
                cells[by, bx] = (BALL, BLUE, 0)
                balls.append((bx, by))
        ck = int(rng.integers(0, 4))
        carry = (EMPTY, 0) if ck == 0 else ((KEY, BALL, BOX)[ck - 1], int(rng.integers(0, 6)))
        rec = list(cells.reshape(-1))
        sc = int(rng.integers(0, max_steps))
        rec += [ax, ay, int(rng.integers(0, 4)), carry[0], carry[1]]
        rec += list(sc.to_bytes(2, "little"))
        rec += list(int(rng.integers(0, 1000)).to_bytes(4, "little"))
        rec += [int(rng.random() < p_prev_done)]
        for bx, by in balls:
            rec += [bx, by]
        if open_edge:
            rec += [int(rng.integers(0, W)), int(rng.integers(0, H))]
        out[e] = rec
    return out
